V=paper_2408_10731_b200/csrc/build/variants
for lay in unit angle; do
python tools/tune_alg1.py --groups 0 --layout $lay 2>&1 | grep tag
for v in g4s4 g2s2m2 g2s3m2 g3s2m2 g6s2 g5s3; do
  TRO_LIB_PATH=$V/libtrajopt_b200_$v.so python tools/tune_alg1.py --groups 0 --layout $lay 2>&1 | grep tag
done
done
for v in g4s4 g2s3m2 g3s2m2; do
  TRO_LIB_PATH=$V/libtrajopt_b200_$v.so python tools/tune_alg1.py --groups 0 --layout unit --dtype f32 2>&1 | grep tag
done
