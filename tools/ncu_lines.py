"""Per-source-line instruction / stall shares of an ncu report (CUDA view)."""
import csv
import subprocess
import sys

rep = sys.argv[1]
n = int(sys.argv[2]) if len(sys.argv) > 2 else 40
txt = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source=cuda,sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(txt.splitlines()))
cur, hdr, out = None, None, []
for r in rows:
    if r and r[0] == "File Path":
        cur = r[1].split("/")[-1]
        continue
    if r and r[0] == "Line No":
        hdr = r
        continue
    if r and r[0].isdigit() and hdr:
        ie, isamp = hdr.index("Instructions Executed"), hdr.index("Warp Stall Sampling (All Samples)")
        try:
            out.append((int(r[ie]), int(r[isamp]), cur, int(r[0]), r[1][:90]))
        except ValueError:
            pass
tot = sum(o[0] for o in out) or 1
ts = sum(o[1] for o in out) or 1
print("instructions", tot, "samples", ts)
for o in sorted(out, reverse=True)[:n]:
    print(f"{o[0] / tot:6.1%} {o[1] / ts:6.1%} {o[2]}:{o[3]} {o[4]}")
