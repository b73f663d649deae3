"""ncu report -> compact JSON summary (per launch) for profiles/."""
import csv
import json
import subprocess
import sys

KEYS = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "smsp__inst_executed.sum", "smsp__inst_executed_pipe_fp64.sum",
        "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active",
        "smsp__issue_active.avg.pct_of_peak_sustained_active",
        "sm__warps_active.avg.pct_of_peak_sustained_active",
        "sm__throughput.avg.pct_of_peak_sustained_elapsed",
        "gpu__compute_memory_throughput.avg.pct_of_peak_sustained_elapsed",
        "launch__registers_per_thread", "launch__grid_size", "launch__block_size",
        "launch__occupancy_limit_registers", "sm__maximum_warps_per_active_cycle_pct",
        "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum"]
rep, out = sys.argv[1], sys.argv[2]
raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True,
                     text=True).stdout
rows = list(csv.reader(raw.splitlines()))
hdr, units = rows[0], rows[1]
launches = []
for r in rows[2:]:
    d = {"kernel": r[hdr.index("Kernel Name")][:120], "id": r[hdr.index("ID")]}
    for k in KEYS:
        if k in hdr:
            i = hdr.index(k)
            d[k] = {"value": r[i], "unit": units[i]}
    st = [(k, float(v)) for k, v in zip(hdr, r)
          if k.startswith("smsp__pcsamp_warps_issue_stalled") and not k.endswith("not_issued")
          and v.replace(".", "").isdigit()]
    tot = sum(v for _, v in st) or 1.0
    d["stall_shares"] = {k.replace("smsp__pcsamp_warps_issue_stalled_", ""): round(v / tot, 4)
                         for k, v in sorted(st, key=lambda t: -t[1])[:8]}
    launches.append(d)
json.dump({"report": rep, "launches": launches}, open(out, "w"), indent=1)
print(out, len(launches), "launches")
