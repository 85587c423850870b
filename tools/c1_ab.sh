# same-box A/B of the C1 in-kernel loop (100 fixed iterations) and the converged solve through solve_single
cd $GRAFT_REPO_ROOT 2>/dev/null || cd /root/repo
for rep in 1 2; do
python tools/c1_loop_time.py
TRO_LIB_PATH=paper_2408_10731_b200/csrc/build/variants/libtrajopt_b200_c1_nocache.so python tools/c1_loop_time.py
done
python - <<'PY'
import time, sys
sys.path.insert(0, ".")
from paper_2408_10731_b200 import scenarios
from paper_2408_10731_b200.solver_single import SingleParams, solve_single
prob = scenarios.c1_problem()
for _ in range(3):
    solve_single(prob, SingleParams())
t0 = time.perf_counter()
for _ in range(20):
    sol = solve_single(prob, SingleParams())
print("converged solve (public API, wall):", (time.perf_counter() - t0) / 20 * 1e3, "ms", sol.iterations, "its")
PY
