# ncu of the Ozaki int8 tensor-core QP GEMM (one launch at C3: 4096 problems) -> gpurun_out/ncu_ozaki.txt
cd $GRAFT_REPO_ROOT 2>/dev/null || cd /root/repo
mkdir -p gpurun_out
ncu --set full --clock-control none --import-source on -k regex:ozaki_gemm -s 2 -c 1 -o gpurun_out/ncu_ozaki -f \
    python tools/ma_qp_ab.py 4096 > gpurun_out/ncu_ozaki.log 2>&1
ncu -i gpurun_out/ncu_ozaki.ncu-rep --page raw --csv > gpurun_out/ncu_ozaki_raw.csv 2>&1
python tools/ncu_summary.py gpurun_out/ncu_ozaki.ncu-rep > gpurun_out/ncu_ozaki.txt 2>&1
python - >> gpurun_out/ncu_ozaki.txt <<'PY'
import csv
rows = list(csv.reader(open("gpurun_out/ncu_ozaki_raw.csv")))
h, v = rows[0], rows[2]
for k, x in zip(h, v):
    if any(t in k for t in ("pipe_tensor", "pipe_tc", "tmem", "uma", "gpu__time_duration.sum", "dram__bytes", "lts__t_bytes.sum", "issue_stalled", "sm__cycles_active.avg", "smsp__cycles_active.avg")):
        print(f"{k:80s} {x}")
PY
rm -f gpurun_out/ncu_ozaki.ncu-rep
