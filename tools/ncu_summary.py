"""One-line-per-launch summary of ncu --set full captures:
python tools/ncu_summary.py a.ncu-rep [b.ncu-rep ...]"""
import csv
import subprocess
import sys

METRICS = ["gpu__time_duration.sum", "launch__grid_size", "launch__block_size",
           "dram__bytes_read.sum", "dram__bytes_write.sum",
           "sm__inst_executed_pipe_tensor_subpipe_dmma.avg.pct_of_peak_sustained_active",
           "sm__ops_path_tensor_src_fp64.avg.pct_of_peak_sustained_elapsed",
           "smsp__average_warps_issue_stalled_barrier_per_issue_active.ratio",
           "smsp__average_warps_issue_stalled_long_scoreboard_per_issue_active.ratio"]
SHORT = ["time", "grid", "block", "dram rd", "dram wr", "DMMA pipe % active", "fp64 tensor ops % peak",
         "barrier stall/issue", "long-scoreboard stall/issue"]

print("| capture | kernel | " + " | ".join(SHORT) + " |")
print("|---|---|" + "---|" * len(SHORT))
for path in sys.argv[1:]:
    out = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv", "--metrics", ",".join(METRICS)],
                         capture_output=True, text=True).stdout
    rows = list(csv.reader(out.splitlines()))
    head, units = rows[0], rows[1]
    ki = head.index("Kernel Name")
    for r in rows[2:]:
        cells = []
        for m in METRICS:
            i = head.index(m)
            cells.append(f"{r[i]} {units[i]}".strip())
        name = r[ki].replace("(anonymous namespace)::", "").replace("unnamed>::", "").split("(")[0]
        print(f"| {path.split('/')[-1]} | {name} | " + " | ".join(cells) + " |")
