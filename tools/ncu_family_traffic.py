"""Per-family DRAM traffic per launch from one `ncu --set full` capture of a
frame (bench.py reads profiles/ncu_summary.json for roofline.traffic), plus
the compact per-launch table.

python tools/ncu_family_traffic.py gpurun_out/frame.ncu-rep profiles/r02_ncu_full.txt profiles/ncu_summary.json"""
import json
import sys

sys.path.insert(0, __file__.rsplit("/", 1)[0])
from ncu_summary import load  # noqa: E402

FAMILY = [("k_conv_plan", "conv_targets"), ("k_conv_targets", "conv_targets"), ("k_conv_dense", "conv_mma"),
          ("k_conv_tc", "conv_mma"), ("k_conv_exact", "conv_mma"), ("k_trunc", "truncate"), ("k_ring_add", "truncate"),
          ("k_maxpool", "pool"), ("k_tile_add", "pool"), ("k_avgpool", "pool"), ("k_densify", "densify"),
          ("k_input", "input_stage"), ("k_warp", "input_stage"), ("k_align", "input_stage"),
          ("k_frame_begin", "frame_begin"), ("k_claims", "claims_reset"), ("k_add", "linear_ops"),
          ("k_upsample", "linear_ops"), ("k_bn", "linear_ops")]


def family(name):
    for key, fam in FAMILY:
        if key in name:
            return fam
    return "other"


rep, txt_out, json_out = sys.argv[1], sys.argv[2], sys.argv[3]
rows = load(rep)
lines, agg = [], {}
for d in rows:
    tr = d.get("dram_rd", 0) + d.get("dram_wr", 0)
    fam = family(d["kernel"])
    a = agg.setdefault(fam, [0.0, 0, 0.0])
    a[0] += tr
    a[1] += 1
    a[2] += d.get("dur_us", 0)
    lines.append(f"{d['kernel'][:40]:40s} {d.get('dur_us', 0):8.1f}us dram={tr / 1e6:8.2f}MB "
                 f"{d.get('dram_pct', 0):5.1f}%dram tensor={d.get('tensor_pct', d.get('tc_pct2', '-'))} "
                 f"warps={d.get('warps_active_pct', '-')} l2hit={d.get('l2_hit', '-')} sm={d.get('sm_thru', '-')} "
                 f"grid={d.get('grid', '-')}")
lines.append("")
for fam, (tr, n, us) in sorted(agg.items()):
    lines.append(f"family {fam:14s} launches {n:3d}  {us:8.1f} us  {tr / 1e6:8.2f} MB  mean {tr / n / 1e6:7.2f} MB/launch")
open(txt_out, "w").write("\n".join(lines) + "\n")
json.dump({"traffic_per_launch": {f: tr / n for f, (tr, n, _) in agg.items()},
           "note": "mean dram__bytes_read.sum + dram__bytes_write.sum per launch of each kernel family, ncu --set full "
                   "over one frame of the default bench workload (cold caches: ncu flushes L2 between launches)",
           "source": txt_out}, open(json_out, "w"), indent=1)
print("\n".join(lines[-len(agg):]))
