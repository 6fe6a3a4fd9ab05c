# aggregate frames/s with S independent camera streams (engines) per GPU
for S in 1 2 4; do
  timeout 600 python bench.py --streams $S --steps 30 --warmup 3 --no-cpu-baseline > gpurun_out/bench_s$S.json 2> gpurun_out/bench_s$S.err
done
python - <<'PY'
import json
out = {}
for S in (1, 2, 4):
    d = json.load(open(f"gpurun_out/bench_s{S}.json"))
    out[f"streams_per_gpu={S}"] = {"frames_per_s": d["value"], "e2e_frames_per_s": d["e2e"]["value"],
                                   "ms_per_step": d["ms_per_step"], "update_rate": d["config"]["update_rate"],
                                   "clocks": d["clocks"]}
json.dump(out, open("gpurun_out/streams.json", "w"), indent=1)
print({k: round(v["frames_per_s"]) for k, v in out.items()})
PY
