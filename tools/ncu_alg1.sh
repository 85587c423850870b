# ncu --set full of one steady-state launch of the Alg. 1 TMA kernel at 16384 members (C5 shape, half layout)
cd $GRAFT_REPO_ROOT 2>/dev/null || cd /root/repo
mkdir -p gpurun_out
TAG=${1:-cur}
LIB=${2:-}
if [ -n "$LIB" ]; then export TRO_LIB_PATH=$LIB; fi
ncu --set full --clock-control none --import-source on -k regex:alg1_tma -s 8 -c 1 -o gpurun_out/ncu_alg1_$TAG -f \
    python tools/tune_alg1.py --members 16384 --iters 10 --layout half > gpurun_out/ncu_alg1_$TAG.log 2>&1
ncu -i gpurun_out/ncu_alg1_$TAG.ncu-rep --page raw --csv > gpurun_out/ncu_alg1_${TAG}_raw.csv 2>&1
