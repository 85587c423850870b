#!/bin/bash
# every bench config once (1 GPU), JSON lines into gpurun_out/final_<cfg>.json
mkdir -p gpurun_out
for cfg in c5 c2 c1 c2alt c3 c4; do
  timeout 900 python bench.py --config $cfg --steps 3 --warmup 3 > gpurun_out/final_$cfg.json 2> gpurun_out/final_$cfg.err
  echo "$cfg rc=$?"; tail -c 400 gpurun_out/final_$cfg.json
done
timeout 600 python bench.py --config c5 --dtype f32 --steps 3 --warmup 3 > gpurun_out/final_c5_f32.json 2> gpurun_out/final_c5_f32.err
echo "c5 f32 rc=$?"
timeout 900 python bench.py --impl reference --steps 1 --warmup 1 > gpurun_out/final_ref_c5.json 2> gpurun_out/final_ref_c5.err
echo "ref rc=$?"; cat gpurun_out/final_ref_c5.json | head -c 300
