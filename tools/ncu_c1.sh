# ncu --set full of the C1 in-kernel loop launch (alg1_kernel MODE 3, 99 iterations of one member)
cd $GRAFT_REPO_ROOT 2>/dev/null || cd /root/repo
mkdir -p gpurun_out
ncu --set full --clock-control none --import-source on -k regex:^alg1_kernel$ -s 3 -c 1 -o gpurun_out/ncu_c1 -f \
    python tools/c1_loop_time.py > gpurun_out/ncu_c1.log 2>&1
{ python tools/ncu_summary.py gpurun_out/ncu_c1.ncu-rep; python tools/ncu_lines.py gpurun_out/ncu_c1.ncu-rep 45; } \
    > gpurun_out/ncu_c1.txt 2>&1
rm -f gpurun_out/ncu_c1.ncu-rep
