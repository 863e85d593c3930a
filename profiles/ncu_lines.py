"""Per-CUDA-line stall samples from an ncu report captured with
--import-source on (kernels compiled with -lineinfo):
    python profiles/ncu_lines.py report.ncu-rep [top]"""
import csv
import subprocess
import sys
from collections import defaultdict

rep = sys.argv[1]
top = int(sys.argv[2]) if len(sys.argv) > 2 else 25
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(out.splitlines()))
f = None
hdr = None
agg = defaultdict(lambda: [0, 0, ""])
stall_cols = []
stalls = defaultdict(lambda: defaultdict(int))
for r in rows:
    if not r:
        continue
    if r[0] == "File Path":
        f = r[1].split("/")[-1]
        continue
    if r[0] == "Line No":
        hdr = r
        stall_cols = [i for i, h in enumerate(hdr) if h.startswith("stall_") and "Not Issued" not in h]
        continue
    if hdr is None or not r[0].isdigit():
        continue
    key = (f, int(r[0]))
    try:
        s = int(r[4] or 0)
        e = int(r[7] or 0)
    except ValueError:
        continue
    agg[key][0] += s
    agg[key][1] += e
    if r[1].strip():
        agg[key][2] = r[1].strip()
    for i in stall_cols:
        try:
            stalls[key][hdr[i][6:]] += int(r[i] or 0)
        except ValueError:
            pass
tot = sum(v[0] for v in agg.values()) or 1
print(f"total samples {tot}")
for key, (s, e, src) in sorted(agg.items(), key=lambda kv: -kv[1][0])[:top]:
    st = sorted(stalls[key].items(), key=lambda kv: -kv[1])[:3]
    print(f"{100 * s / tot:5.1f}% {key[0]}:{key[1]:<5} inst {e:<8} {src[:70]:<70} {st}")
