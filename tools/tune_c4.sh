#!/bin/bash
# PRIEST projection launch time (C4 shape) for the default library and each variant argument
V=paper_2408_10731_b200/csrc/build/variants
run() { python bench.py --config c4 --steps 1 --warmup 1 --no-cpu-baseline --no-e2e 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$1', round(d['roofline']['avg_launch_ms'],3), round(d['roofline']['frac'],3))"; }
run default
for v in "$@"; do TRO_LIB_PATH=$V/libtrajopt_b200_$v.so run $v; done
