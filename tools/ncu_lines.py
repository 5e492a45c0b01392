"""Per-source-line instruction and stall-sample totals from an ncu report (cuda,sass view)."""
import collections
import csv
import subprocess
import sys

rep = sys.argv[1]
kf = sys.argv[2] if len(sys.argv) > 2 else ""
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                     capture_output=True, text=True).stdout.splitlines()
fname, func, hdr = None, None, None
inst = collections.Counter()
samp = collections.Counter()
text = {}
for row in csv.reader(out):
    if not row:
        continue
    if row[0] == "File Path":
        fname = row[1].split("/")[-1]
        continue
    if row[0] == "Function Name":
        func = row[1]
        continue
    if row[0] == "Line No":
        hdr = row
        continue
    if hdr is None or (kf and kf not in (func or "")):
        continue
    try:
        ln = int(row[0])
    except ValueError:
        continue
    key = (fname, ln)
    text[key] = row[1][:90]
    try:
        inst[key] += int(row[hdr.index("Instructions Executed")] or 0)
        samp[key] += int(row[hdr.index("Warp Stall Sampling (All Samples)")] or 0)
    except (ValueError, IndexError):
        pass
tot_i = sum(inst.values()) or 1
tot_s = sum(samp.values()) or 1
print(f"total warp instructions {tot_i}, samples {tot_s}")
for key, v in sorted(inst.items(), key=lambda kv: -kv[1])[:int(sys.argv[3]) if len(sys.argv) > 3 else 30]:
    print(f"{100*v/tot_i:5.1f}% inst {100*samp[key]/tot_s:5.1f}% stall  {key[0]}:{key[1]}  {text[key]}")
