"""Summarize an ncu report: key raw metrics, stall mix, opcode histogram, top stall sites."""
import collections
import csv
import subprocess
import sys

rep = sys.argv[1]
kfilter = sys.argv[2] if len(sys.argv) > 2 else None
raw = list(csv.reader(subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout.splitlines()))
h = raw[0]
want = ["Kernel Name", "gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "sm__warps_active.avg.pct_of_peak_sustained_active",
        "launch__registers_per_thread", "launch__occupancy_limit_shared_mem", "launch__occupancy_limit_registers",
        "launch__grid_size", "launch__block_size", "launch__shared_mem_per_block_dynamic", "smsp__inst_executed.sum",
        "smsp__thread_inst_executed.sum", "smsp__issue_active.avg.pct_of_peak_sustained_active",
        "sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active", "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum",
        "lts__t_bytes.sum"]
for r in raw[2:]:
    if kfilter and kfilter not in r[h.index("Kernel Name")]:
        continue
    for w in want:
        if w in h:
            print(f"  {w:60s} {r[h.index(w)]}")
    print("  ---")
src = list(csv.reader(subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv"], capture_output=True, text=True).stdout.splitlines()))
blocks, cur = [], None
for row in src:
    if row and row[0] == "Kernel Name":
        cur = {"name": row[1], "rows": []}
        blocks.append(cur)
        continue
    if row and row[0] == "Address":
        cur["hdr"] = row
        continue
    if cur is not None and row and row[0].startswith("0x"):
        cur["rows"].append(row)
for b in blocks:
    if kfilter and kfilter not in b["name"]:
        continue
    hd = b["hdr"]
    iS, iI, iT = hd.index("Warp Stall Sampling (All Samples)"), hd.index("Instructions Executed"), hd.index("Thread Instructions Executed")
    cols = [c for c in hd if c.startswith("stall_") and "Not Issued" not in c]
    idx = [hd.index(c) for c in cols]
    rows = b["rows"]
    T = sum(float(x[iS] or 0) for x in rows) or 1
    tot = collections.Counter()
    for x in rows:
        for c, i in zip(cols, idx):
            tot[c] += float(x[i] or 0)
    print(b["name"], "samples", T)
    print("  stalls:", ", ".join(f"{c[6:]} {100 * v / T:.1f}%" for c, v in tot.most_common(8)))
    c, ct = collections.Counter(), collections.Counter()
    for x in rows:
        ins = x[1].strip().split()
        op = ins[1] if ins[0].startswith("@") else ins[0]
        op = op.split(".")[0]
        c[op] += float(x[iI] or 0)
        ct[op] += float(x[iT] or 0)
    ti = sum(c.values())
    print(f"  warp-inst {ti:.0f}  thread-inst {sum(ct.values()):.0f}  avg lanes {sum(ct.values()) / max(ti, 1):.1f}")
    print("  ", "  ".join(f"{k}:{100 * v / ti:.1f}%/{ct[k] / max(v, 1):.0f}l" for k, v in c.most_common(14)))
    for x in sorted(rows, key=lambda x: -float(x[iS] or 0))[:12]:
        top = max(zip(cols, idx), key=lambda ci: float(x[ci[1]] or 0))
        print(f"  {100 * float(x[iS]) / T:5.1f}% {x[iI]:>9} {top[0][6:]:14s} {x[1].strip()[:70]}")
