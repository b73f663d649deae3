"""Summarise an ncu report: duration, issue, stalls, instruction mix (SASS opcode counts)."""
import csv
import subprocess
import sys
from collections import Counter

rep = sys.argv[1]
raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
r = list(csv.reader(raw.splitlines()))
h, v = r[0], r[2]
keys = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "smsp__inst_executed.sum", "smsp__issue_active.avg.pct_of_peak_sustained_active",
        "sm__warps_active.avg.pct_of_peak_sustained_active",
        "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active",
        "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum", "launch__registers_per_thread",
        "launch__grid_size", "sm__cycles_elapsed.avg"]
for k, x in zip(h, v):
    if k in keys:
        print(f"{k:70s} {x}")
st = [(k, x) for k, x in zip(h, v) if k.startswith("smsp__pcsamp_warps_issue_stalled") and not k.endswith("not_issued")]
tot = sum(float(x) for _, x in st if x.replace('.', '').isdigit())
for k, x in sorted(st, key=lambda t: -float(t[1]) if t[1].replace('.', '').isdigit() else 0)[:8]:
    print(f"  stall {k.replace('smsp__pcsamp_warps_issue_stalled_', ''):28s} {float(x) / tot:6.1%}")
sass = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source=sass"],
                      capture_output=True, text=True).stdout
rows = list(csv.reader(sass.splitlines()))
hh = rows[1]
ia = hh.index("Instructions Executed")
c = Counter()
for row in rows[2:]:
    if not row[ia].isdigit():
        continue
    t = row[1].split()
    if not t:
        continue
    op = t[1] if t[0].startswith("@") else t[0]
    c[op.split(".")[0]] += int(row[ia])
tot_i = sum(c.values())
print("SASS instructions executed:", tot_i, " static:", len(rows) - 2)
print("  " + ", ".join(f"{op} {n / tot_i:.1%}" for op, n in c.most_common(14)))
