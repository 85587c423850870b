#!/bin/bash
# fp32 Alg. 1 at 3 CTAs/SM (80-register cap) vs the base 2, full C5 size
V=paper_2408_10731_b200/csrc/build/variants
for lib in base m3 m3s3 base; do
  if [ $lib = base ]; then unset TRO_LIB_PATH; else export TRO_LIB_PATH=$V/libtrajopt_b200_$lib.so; fi
  out=$(timeout 300 python bench.py --config c5 --dtype f32 --steps 2 --warmup 3 --no-cpu-baseline --no-e2e 2>/dev/null | tail -1)
  echo "$lib $(echo "$out" | python -c 'import json,sys; d=json.loads(sys.stdin.read()); r=d["roofline"]; print(round(r["avg_launch_ms"],3), round(r["frac"],4), d["clocks"]["sm_mhz"])' 2>&1)"
done
