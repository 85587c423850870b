V=paper_2408_10731_b200/csrc/build/variants
for lay in angle unit; do
python tools/tune_alg1.py --groups 0 --layout $lay 2>&1 | grep tag
for v in g6s2 g4 g8s1; do
  TRO_LIB_PATH=$V/libtrajopt_b200_$v.so python tools/tune_alg1.py --groups 0 --layout $lay 2>&1 | grep tag
done
python tools/tune_alg1.py --groups 0 --dtype f32 --layout $lay 2>&1 | grep tag
TRO_LIB_PATH=$V/libtrajopt_b200_g6s2.so python tools/tune_alg1.py --groups 0 --dtype f32 --layout $lay 2>&1 | grep tag
done
