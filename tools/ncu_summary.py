"""Summarise ncu --set full reports (raw page) into a compact per-launch table."""
import csv, io, json, subprocess, sys

KEYS = {
    "dur_us": "gpu__time_duration.sum",
    "dram_rd": "dram__bytes_read.sum",
    "dram_wr": "dram__bytes_write.sum",
    "dram_pct": "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
    "tensor_pct": "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed",
    "tc_pct2": "sm__pipe_tc_cycles_active.avg.pct_of_peak_sustained_elapsed",
    "warps_active_pct": "sm__warps_active.avg.pct_of_peak_sustained_active",
    "regs": "launch__registers_per_thread",
    "l2_hit": "lts__t_sector_hit_rate.pct",
    "sm_thru": "sm__throughput.avg.pct_of_peak_sustained_elapsed",
    "l1_bytes": "l1tex__t_bytes.sum",
    "lts_bytes": "lts__t_bytes.sum",
    "grid": "launch__grid_size",
}


def load(path):
    if path.endswith(".csv"):  # an exported raw page (ncu -i rep --page raw --csv)
        out = open(path).read()
    else:
        out = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr, units = rows[0], rows[1]
    res = []
    for r in rows[2:]:
        d = {"kernel": r[hdr.index("Kernel Name")][:48]}
        for k, m in KEYS.items():
            if m in hdr:
                i = hdr.index(m)
                v = r[i].replace(",", "")
                try:
                    v = float(v)
                except ValueError:
                    pass
                u = units[i]
                if k == "dur_us":
                    v = v / 1e3 if u == "ns" else (v * 1e3 if u == "ms" else v)
                if k in ("dram_rd", "dram_wr", "l1_bytes", "lts_bytes") and isinstance(v, float):
                    v = v * {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}.get(u, 1)
                d[k] = v
        res.append(d)
    return res


if __name__ == "__main__":
    allr = {}
    for p in sys.argv[1:]:
        rs = load(p)
        allr[p] = rs
        for d in rs:
            tr = (d.get("dram_rd", 0) + d.get("dram_wr", 0)) / 1e6
            print(f"{d['kernel'][:34]:34s} {d.get('dur_us',0):8.1f}us dram={tr:8.2f}MB {d.get('dram_pct',0):5.1f}%dram "
                  f"tc={d.get('tensor_pct', d.get('tc_pct2', '-'))} warps={d.get('warps_active_pct','-')} "
                  f"l2hit={d.get('l2_hit','-')} sm={d.get('sm_thru','-')} grid={d.get('grid','-')}")
