"""Key metrics of the first kernel in an ncu report."""
import csv
import io
import subprocess
import sys

rep = sys.argv[1]
det = subprocess.run(["ncu", "-i", rep, "--page", "details", "--csv"], capture_output=True, text=True).stdout
keys = {"Duration", "Registers Per Thread", "Achieved Occupancy", "Executed Ipc Active", "Issue Slots Busy",
        "Warp Cycles Per Issued Instruction", "Executed Instructions", "DRAM Throughput", "Memory Throughput"}
seen = set()
for row in csv.reader(io.StringIO(det)):
    if len(row) > 4 and row[-4] in keys and row[-4] not in seen:
        seen.add(row[-4])
        print(f"{row[-4]:40s} {row[-2]:>14s} {row[-3]}")
raw = list(csv.reader(io.StringIO(subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True,
                                                 text=True).stdout)))
h, v = raw[0], raw[2]
for k, x in zip(h, v):
    if k in ("sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active",
             "sm__inst_executed_pipe_lsu.sum.pct_of_peak_sustained_active",
             "sm__inst_executed_pipe_alu.sum.pct_of_peak_sustained_active",
             "sm__inst_executed_pipe_xu.sum.pct_of_peak_sustained_active",
             "dram__bytes_read.sum", "dram__bytes_write.sum", "gpu__time_duration.sum"):
        print(f"{k:70s} {x}")
    elif "average_warps_issue_stalled" in k and k.endswith("per_issue_active.ratio"):
        try:
            if float(x) > 0.3:
                print(f"{k:70s} {x}")
        except ValueError:
            pass
