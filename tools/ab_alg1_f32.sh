# same-box A/B of the fp32 Alg. 1 TMA kernel variants at the C5 shape (32768 members, n_o 100)
cd $GRAFT_REPO_ROOT 2>/dev/null || cd /root/repo
for rep in 1 2; do
for n in f_g4m1s6 f2_def f2_g2m2; do
for lay in unit half; do
  TRO_LIB_PATH=paper_2408_10731_b200/csrc/build/variants/libtrajopt_b200_$n.so python tools/tune_alg1.py --members 32768 --iters 20 --layout $lay --dtype f32 --tag $n 2>&1 | tail -1
done
done
done
