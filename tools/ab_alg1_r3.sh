# same-box A/B: current library vs the previous variants, C5 shape (32768 members, n_o 100, half layout)
cd $GRAFT_REPO_ROOT 2>/dev/null || cd /root/repo
for rep in 1 2; do
python tools/tune_alg1.py --members 32768 --iters 20 --layout half --tag cur 2>&1 | tail -1
TRO_LIB_PATH=paper_2408_10731_b200/csrc/build/variants/libtrajopt_b200_n2_rcp1.so python tools/tune_alg1.py --members 32768 --iters 20 --layout half --tag prev 2>&1 | tail -1
python tools/tune_alg1.py --members 32768 --iters 20 --layout half --dtype f32 --tag cur 2>&1 | tail -1
TRO_LIB_PATH=paper_2408_10731_b200/csrc/build/variants/libtrajopt_b200_f2_def.so python tools/tune_alg1.py --members 32768 --iters 20 --layout half --dtype f32 --tag prev 2>&1 | tail -1
done
