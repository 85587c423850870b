cd $GRAFT_REPO_ROOT 2>/dev/null || cd /root/repo
mkdir -p gpurun_out
bash tools/ncu_alg1.sh r2final f64 0
bash tools/ncu_alg1.sh r2finalf32 f32 0
# launch list of the C5 bench command (first 400 launches, 16384-member shard of the same recipe)
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/r2_launches_c5.csv \
    python bench.py --steps 1 --warmup 0 --members 16384 --no-cpu-baseline --no-e2e > gpurun_out/r2_launches_c5.log 2>&1
# multi-agent element kernel, one launch at C3
ncu --set full --clock-control none --import-source on -k regex:^ma_kernel$ -s 20 -c 1 -o gpurun_out/ncu_ma -f \
    python tools/ma_ab.py > gpurun_out/ncu_ma.log 2>&1
{ python tools/ncu_summary.py gpurun_out/ncu_ma.ncu-rep; python tools/ncu_lines.py gpurun_out/ncu_ma.ncu-rep 50; } > gpurun_out/ncu_ma.txt 2>&1
rm -f gpurun_out/ncu_ma.ncu-rep
