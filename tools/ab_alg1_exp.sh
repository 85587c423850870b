cd $GRAFT_REPO_ROOT 2>/dev/null || cd /root/repo
mkdir -p gpurun_out
for rep in 1 2; do
for n in base nopro notrk rcp1 all3 s4; do
  TRO_LIB_PATH=paper_2408_10731_b200/csrc/build/variants/libtrajopt_b200_$n.so python tools/tune_alg1.py --members 32768 --iters 20 --layout half --tag $n 2>&1 | tail -1
done
done
