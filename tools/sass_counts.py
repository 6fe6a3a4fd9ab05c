"""Per-kernel SASS instruction counts of libdfx_b200.so (cuobjdump -sass):
the evidence that the convs issue tcgen05 MMAs (UTCHMMA) with TMEM traffic
(LDTM / STTM) and bulk copies (UBLKCP), and how each kernel moves memory.
python tools/sass_counts.py > profiles/r02_sass_counts.json"""
import collections
import json
import re
import subprocess
import sys

lib = sys.argv[1] if len(sys.argv) > 1 else "paper_2210_09887_b200/libdfx_b200.so"
txt = subprocess.run(["cuobjdump", "-sass", lib], capture_output=True, text=True).stdout
KEYS = ["UTCHMMA", "UTCQMMA", "UTCBAR", "LDTM", "STTM", "UBLKCP", "UBLKPF", "UTMALDG", "UTMASTG", "LDGSTS", "LDG",
        "STG", "ATOMG", "REDG", "SHFL", "MATCH", "REDUX", "SYNCS", "FADD", "FFMA", "FMNMX"]
out = {}
for part in re.split(r"\n\s*Function : ", txt)[1:]:
    mangled = part.split("\n", 1)[0].strip()
    name = subprocess.run(["c++filt", mangled], capture_output=True, text=True).stdout.strip()
    name = name.replace("dfx::(anonymous namespace)::", "").replace("(anonymous namespace)::", "")
    name = re.sub(r"\(.*", "", name)
    ops = re.findall(r"/\*[0-9a-f]{4,}\*/\s+(?:@!?U?P[T0-9]+\s+)?([A-Z][A-Z0-9_]*)", part)
    c = collections.Counter(ops)
    row = {k: c[k] for k in KEYS if c.get(k)}
    row["instructions"] = sum(c.values())
    out[name] = row
print(json.dumps(out, indent=1, sort_keys=True))
