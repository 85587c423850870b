# ncu of the multi-agent element kernel (C3, 4096 problems) with per-source-line stall samples
cd $GRAFT_REPO_ROOT 2>/dev/null || cd /root/repo
mkdir -p gpurun_out
timeout 300 python tools/tune_ma.py --problems 4096 --iters 10 > gpurun_out/ma_time.json 2>&1
ncu --set full --clock-control none --import-source on -k regex:ma_kernel -s 6 -c 1 -o gpurun_out/ncu_ma -f \
    python tools/tune_ma.py --problems 4096 --iters 3 > gpurun_out/ncu_ma.log 2>&1
python tools/ncu_summary.py gpurun_out/ncu_ma.ncu-rep > gpurun_out/ncu_ma.txt 2>&1
python tools/ncu_lines.py gpurun_out/ncu_ma.ncu-rep 60 > gpurun_out/ncu_ma_lines.txt 2>&1
python tools/ncu_lines_smem.py gpurun_out/ncu_ma.ncu-rep 40 > gpurun_out/ncu_ma_smem.txt 2>&1
ncu -i gpurun_out/ncu_ma.ncu-rep --page raw --csv > gpurun_out/ncu_ma_raw.csv 2>&1
python - >> gpurun_out/ncu_ma.txt <<'PY'
import csv
rows = list(csv.reader(open("gpurun_out/ncu_ma_raw.csv")))
h, v = rows[0], rows[2]
for k, x in zip(h, v):
    if any(t in k for t in ("shared_op", "mem_shared", "bank", "l1tex__throughput", "lsu_mem", "l1tex__data_pipe_lsu",
                            "sm__warps_active", "launch__occupancy_limit", "smsp__thread_inst_executed_per_inst",
                            "dmma", "pipe_tensor", "pipe_fp64")):
        print(f"{k:90s} {x}")
PY
rm -f gpurun_out/ncu_ma.ncu-rep gpurun_out/ncu_ma_raw.csv
