"""Per-kernel times of the last frame in an ncu launch-list CSV."""
import csv, sys
rows = [r for r in csv.reader(open(sys.argv[1] if len(sys.argv) > 1 else 'gpurun_out/launches.csv')) if len(r) > 10][1:]
idx = [i for i, r in enumerate(rows) if 'k_frame_begin' in r[4]] or [i for i, r in enumerate(rows) if 'k_claims' in r[4]]
s = idx[-1]
tot = 0
for r in rows[s:]:
    v = float(r[14]) / 1e3
    tot += v
    print(f"{v:9.1f}us grid={r[8]:14s} blk={r[7]:12s} {r[4][:70]}")
print(f"total {tot:.1f} us, {len(rows) - s} launches")
