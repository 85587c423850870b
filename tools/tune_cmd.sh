V=paper_2408_10731_b200/csrc/build/variants
python tools/tune_alg1.py --groups 2,3,4,5 2>&1 | grep tag
for v in u1 u1b320 u2b320 u1b256 u1b416; do
  TRO_LIB_PATH=$V/libtrajopt_b200_$v.so python tools/tune_alg1.py --groups 2,3,4,5 2>&1 | grep tag
done
python tools/tune_alg1.py --groups 2,4,5 --dtype f32 2>&1 | grep tag
