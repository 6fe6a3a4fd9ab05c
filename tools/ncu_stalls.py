"""Top stalled SASS instructions of one launch in an ncu report (source page)."""
import csv, io, subprocess, sys
rep, skip = sys.argv[1], int(sys.argv[2]) if len(sys.argv) > 2 else 0
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--launch-skip", str(skip), "--launch-count", "1"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
hdr = None; data = []; seen = set()
for r in rows:
    if 'Address' in r and 'Source' in r:
        hdr = r; continue
    if hdr and len(r) == len(hdr) and r[0].startswith('0x') and r[0] not in seen:
        seen.add(r[0]); data.append(r)
si = hdr.index('Warp Stall Sampling (All Samples)'); src = hdr.index('Source')
f = lambda r: float(r[si] or 0)
tot = sum(map(f, data))
idx = {r[0]: i for i, r in enumerate(data)}
for r in sorted(data, key=lambda r: -f(r))[:int(sys.argv[3]) if len(sys.argv) > 3 else 25]:
    i = idx[r[0]]
    ctx = " | ".join(d[src].strip()[:40] for d in data[max(0, i - 3):i])
    print(f"{f(r) / tot * 100:5.1f}% {r[0][-5:]} {r[src].strip()[:60]:60s}  <- {ctx}")
