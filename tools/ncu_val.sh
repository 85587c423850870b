# ncu of the batched validation kernel (val config: 131072 C5 trajectories x 100 obstacles), per-line samples
cd $GRAFT_REPO_ROOT 2>/dev/null || cd /root/repo
mkdir -p gpurun_out
ncu --set full --import-source on --clock-control none -k regex:validate_kernel -s 3 -c 1 -o gpurun_out/ncu_val -f \
    python bench.py --config val --steps 1 --warmup 3 > gpurun_out/ncu_val.log 2>&1
python tools/ncu_summary.py gpurun_out/ncu_val.ncu-rep > gpurun_out/ncu_val.txt 2>&1
python tools/ncu_lines.py gpurun_out/ncu_val.ncu-rep 40 > gpurun_out/ncu_val_lines.txt 2>&1
python tools/ncu_lines_smem.py gpurun_out/ncu_val.ncu-rep 12 > gpurun_out/ncu_val_smem.txt 2>&1
rm -f gpurun_out/ncu_val.ncu-rep
