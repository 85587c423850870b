#!/bin/bash
# time the Alg. 2 device loop for the default library and every variant given as arguments
V=paper_2408_10731_b200/csrc/build/variants
echo -n "default: "; python tools/b2_quick.py 2>&1 | grep "device loop"
for v in "$@"; do
  echo -n "$v: "; TRO_LIB_PATH=$V/libtrajopt_b200_$v.so python tools/b2_quick.py 2>&1 | grep "device loop"
done
