# ncu of the Alg. 2 iterate kernel (C2-alt, launch 41) + per-source-line stall samples
cd $GRAFT_REPO_ROOT 2>/dev/null || cd /root/repo
mkdir -p gpurun_out
ncu --set full --import-source on --clock-control none -k regex:b2_kernel --launch-skip 40 --launch-count 1 \
    -o gpurun_out/ncu_b2 -f python tools/b2_profile.py > gpurun_out/ncu_b2.log 2>&1
python tools/ncu_summary.py gpurun_out/ncu_b2.ncu-rep > gpurun_out/ncu_b2.txt 2>&1
python tools/ncu_lines.py gpurun_out/ncu_b2.ncu-rep 80 > gpurun_out/ncu_b2_lines.txt 2>&1
rm -f gpurun_out/ncu_b2.ncu-rep
