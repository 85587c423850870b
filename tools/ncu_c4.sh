# ncu of the PRIEST projection kernel (C4: 16384 samples x 100 spheres x n_p 100 x 30 inner its), per-line samples
cd $GRAFT_REPO_ROOT 2>/dev/null || cd /root/repo
mkdir -p gpurun_out
ncu --set full --import-source on --clock-control none -k regex:priest_project -s 2 -c 1 -o gpurun_out/ncu_c4 -f \
    python bench.py --config c4 --steps 1 --warmup 3 > gpurun_out/ncu_c4.log 2>&1
python tools/ncu_summary.py gpurun_out/ncu_c4.ncu-rep > gpurun_out/ncu_c4.txt 2>&1
python tools/ncu_lines.py gpurun_out/ncu_c4.ncu-rep 40 > gpurun_out/ncu_c4_lines.txt 2>&1
python tools/ncu_lines_smem.py gpurun_out/ncu_c4.ncu-rep 25 > gpurun_out/ncu_c4_smem.txt 2>&1
rm -f gpurun_out/ncu_c4.ncu-rep
