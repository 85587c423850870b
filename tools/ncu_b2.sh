#!/bin/bash
# usage: tools/ncu_b2.sh NAME  -> gpurun_out/NAME.ncu-rep (iterate kernel, launch 41)
ncu --set full --import-source on --clock-control none -k regex:b2_kernel --launch-skip 40 --launch-count 1 \
    -o gpurun_out/$1 python tools/b2_profile.py > gpurun_out/$1.log 2>&1
tail -1 gpurun_out/$1.log
