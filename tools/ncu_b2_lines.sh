# ncu of the Alg. 2 iterate kernel (C2-alt, launch 41) + per-source-line stall samples
cd $GRAFT_REPO_ROOT 2>/dev/null || cd /root/repo
mkdir -p gpurun_out
ncu --set full --import-source on --clock-control none -k regex:b2_kernel --launch-skip 40 --launch-count 1 \
    -o gpurun_out/ncu_b2 -f python tools/b2_profile.py > gpurun_out/ncu_b2.log 2>&1
python tools/ncu_summary.py gpurun_out/ncu_b2.ncu-rep > gpurun_out/ncu_b2.txt 2>&1
python tools/ncu_lines.py gpurun_out/ncu_b2.ncu-rep 80 > gpurun_out/ncu_b2_lines.txt 2>&1
python tools/ncu_lines_smem.py gpurun_out/ncu_b2.ncu-rep 12 > gpurun_out/ncu_b2_smem.txt 2>&1
ncu -i gpurun_out/ncu_b2.ncu-rep --page raw --csv > gpurun_out/ncu_b2_raw.csv 2>&1
python - >> gpurun_out/ncu_b2.txt <<'PY'
import csv
rows = list(csv.reader(open("gpurun_out/ncu_b2_raw.csv")))
h, v = rows[0], rows[2]
for k, x in zip(h, v):
    if any(t in k for t in ("hit_rate", "l1tex__t_sectors_pipe_lsu_mem_global_op_ld.sum", "lts__t_sectors_srcunit_tex_op_read.sum",
                            "launch__shared_mem", "launch__occupancy", "sm__warps_active.avg.pct", "l1tex__data_pipe_lsu_wavefronts.avg.pct")):
        print(f"{k:90s} {x}")
PY
rm -f gpurun_out/ncu_b2.ncu-rep gpurun_out/ncu_b2_raw.csv
