#!/bin/bash
# DRAM traffic of each config's dominant kernel (one launch each), for bench.py's roofline.traffic.
# usage (on the GPU box): tools/ncu_traffic.sh  -> gpurun_out/traffic_*.csv
M="dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum"
mkdir -p gpurun_out
ncu --metrics $M --clock-control none -k regex:priest_project_kernel --launch-skip 4 --launch-count 1 --csv \
    python bench.py --config c4 --steps 1 --warmup 1 --no-cpu-baseline > gpurun_out/traffic_c4.csv 2>/dev/null
ncu --metrics $M --clock-control none -k regex:ma_kernel --launch-skip 30 --launch-count 1 --csv \
    python bench.py --config c3 --steps 1 --warmup 1 --no-cpu-baseline > gpurun_out/traffic_c3.csv 2>/dev/null
ncu --metrics $M --clock-control none -k regex:b2_kernel --launch-skip 60 --launch-count 1 --csv \
    python bench.py --config c2alt --steps 1 --warmup 1 --no-cpu-baseline > gpurun_out/traffic_c2alt.csv 2>/dev/null
ncu --metrics $M --clock-control none -k regex:alg1_tma_kernel --launch-skip 30 --launch-count 1 --csv \
    python bench.py --config c2 --steps 1 --warmup 1 --no-cpu-baseline > gpurun_out/traffic_c2.csv 2>/dev/null
grep -h "dram__bytes\|gpu__time" gpurun_out/traffic_*.csv | cut -c1-200
# §8(f) lines (validation, MPC fleet) and the fp32 Alg. 1 build at the C5 shape (16384 members)
ncu --metrics $M --clock-control none -k regex:validate_kernel --launch-skip 3 --launch-count 1 --csv \
    python bench.py --config val --steps 1 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/traffic_val.csv 2>/dev/null
ncu --metrics $M --clock-control none -k regex:alg1_tma_kernel --launch-skip 200 --launch-count 1 --csv \
    python bench.py --config mpc --steps 1 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/traffic_mpc.csv 2>/dev/null
ncu --metrics $M,smsp__inst_executed.sum,sm__inst_executed_pipe_fma.avg.pct_of_peak_sustained_active,smsp__issue_active.avg.pct_of_peak_sustained_active \
    --clock-control none -k regex:alg1_tma_kernel --launch-skip 30 --launch-count 1 --csv \
    python bench.py --config c5 --dtype f32 --members 16384 --steps 1 --warmup 3 --no-cpu-baseline --no-e2e \
    > gpurun_out/traffic_c5_f32.csv 2>/dev/null
grep -h "dram__bytes\|gpu__time" gpurun_out/traffic_*.csv | cut -c1-200
