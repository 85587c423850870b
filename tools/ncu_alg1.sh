# ncu --set full of one steady-state launch of the Alg. 1 TMA kernel at 16384 members (C5 shape, half layout);
# leaves gpurun_out/ncu_alg1_<tag>.{ncu-rep,txt}: the report and its summary (tools/ncu_summary.py, ncu_lines.py)
cd $GRAFT_REPO_ROOT 2>/dev/null || cd /root/repo
mkdir -p gpurun_out
TAG=${1:-cur}
DT=${2:-f64}
KEEP=${3:-1}
ncu --set full --clock-control none --import-source on -k regex:alg1_tma -s 8 -c 1 -o gpurun_out/ncu_alg1_$TAG -f \
    python tools/tune_alg1.py --members 16384 --iters 10 --layout half --dtype $DT > gpurun_out/ncu_alg1_$TAG.log 2>&1
{ python tools/ncu_summary.py gpurun_out/ncu_alg1_$TAG.ncu-rep; python tools/ncu_lines.py gpurun_out/ncu_alg1_$TAG.ncu-rep 40; } \
    > gpurun_out/ncu_alg1_$TAG.txt 2>&1
if [ "$KEEP" = "0" ]; then rm -f gpurun_out/ncu_alg1_$TAG.ncu-rep; fi
