#!/bin/bash
# fp32 Alg. 1 A/B at the full C5 size: stage count / rows per stage / layout
mkdir -p gpurun_out
V=paper_2408_10731_b200/csrc/build/variants
for lib in base s5 s6 g3; do
  for lay in unit half; do
    if [ $lib = base ]; then unset TRO_LIB_PATH; else export TRO_LIB_PATH=$V/libtrajopt_b200_$lib.so; fi
    out=$(timeout 300 python bench.py --config c5 --dtype f32 --layout $lay --steps 2 --warmup 3 --no-cpu-baseline --no-e2e 2>/dev/null | tail -1)
    echo "$lib $lay $(echo "$out" | python -c 'import json,sys; d=json.loads(sys.stdin.read()); r=d["roofline"]; print(round(r["avg_launch_ms"],3), round(r["frac"],4), d["clocks"]["sm_mhz"])' 2>&1)"
  done
done
