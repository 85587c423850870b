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
