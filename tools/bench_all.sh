#!/bin/bash
# every bench config once (1 GPU), JSON lines into gpurun_out/final_<cfg>.json, then the reference arms
cd $GRAFT_REPO_ROOT 2>/dev/null || cd /root/repo
mkdir -p gpurun_out
for cfg in c5 c2 c1 c2alt c3 c4 val mpc; do
  timeout 900 python bench.py --config $cfg --steps 3 --warmup 3 > gpurun_out/final_$cfg.json 2> gpurun_out/final_$cfg.err
  echo "$cfg rc=$?"; tail -c 300 gpurun_out/final_$cfg.json; echo
done
timeout 600 python bench.py --config c5 --dtype f32 --steps 3 --warmup 3 > gpurun_out/final_c5_f32.json 2> gpurun_out/final_c5_f32.err
echo "c5 f32 rc=$?"
for cfg in c5 mpc; do
  timeout 900 python bench.py --impl reference --config $cfg --steps 1 --warmup 1 > gpurun_out/final_ref_$cfg.json 2> gpurun_out/final_ref_$cfg.err
  echo "ref $cfg rc=$?"; head -c 300 gpurun_out/final_ref_$cfg.json; echo
done
