"""Top SASS lines of one kernel in an ncu report by stall samples, with the
instruction mix: python profiles/ncu_hot.py REP KERNEL_REGEX [N]"""
import csv
import subprocess
import sys

rep, kern = sys.argv[1], sys.argv[2]
n = int(sys.argv[3]) if len(sys.argv) > 3 else 40
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "-k", "regex:" + kern,
                      "--print-source", "sass"], capture_output=True, text=True).stdout
rows = list(csv.reader(out.splitlines()))
hi = [i for i, r in enumerate(rows) if r and r[0] == "Address"][0]
h = rows[hi]
body = [r for r in rows[hi + 1:] if len(r) == len(h) and r[0] != "Address"]
si, ii, src = h.index("Warp Stall Sampling (All Samples)"), h.index("Instructions Executed"), h.index("Source")
tot = sum(int(r[si] or 0) for r in body)
tot_i = sum(int(r[ii] or 0) for r in body)
print(f"samples {tot}, warp instructions {tot_i}")
mix = {}
for r in body:
    op = r[src].split()[0] if r[src].split() else "?"
    if op.startswith("@"):
        op = r[src].split()[1]
    op = op.split(".")[0]
    mix[op] = mix.get(op, 0) + int(r[ii] or 0)
print("mix:", ", ".join(f"{k} {v}" for k, v in sorted(mix.items(), key=lambda x: -x[1])[:25]))
for r in sorted(body, key=lambda r: -int(r[si] or 0))[:n]:
    print(f"{int(r[si] or 0):6d} {int(r[ii] or 0):9d}  {r[0][-5:]}  {r[src][:90]}")
