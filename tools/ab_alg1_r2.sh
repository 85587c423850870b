# same-box A/B of Alg. 1 TMA-kernel variants at the C5 shape (32768 members, n_o 100, half layout)
cd $GRAFT_REPO_ROOT 2>/dev/null || cd /root/repo
for rep in 1 2; do
for n in base all3 n2_g4s4 n2_g4s5 n2_rcp1 n2_g2m2; do
  TRO_LIB_PATH=paper_2408_10731_b200/csrc/build/variants/libtrajopt_b200_$n.so python tools/tune_alg1.py --members 32768 --iters 20 --layout half --tag $n 2>&1 | tail -1
done
done
