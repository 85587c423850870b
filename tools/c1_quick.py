"""C1 timings: device loop (per-launch vs in-kernel loop) and the drop-in API."""
import os
import sys
import time

sys.path.insert(0, os.path.join(os.path.dirname(os.path.abspath(__file__)), ".."))
import torch  # noqa: E402

from paper_2408_10731_b200 import scenarios, solver_single  # noqa: E402
from paper_2408_10731_b200 import _alg1  # noqa: E402

prob = scenarios.c1_problem()
for loop in (False, True):
    params = solver_single.SingleParams(max_iter=100, tol=0.0)
    eng = solver_single._engine_for(prob, params, max_hist=100)
    for rep in range(3):
        eng.reset_schedule()
        eng.cold_init()
        torch.cuda.synchronize()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        eng.run(100, use_graph=True, loop=loop)
        b.record()
        torch.cuda.synchronize()
    print(f"loop={loop}: {a.elapsed_time(b):.3f} ms / 100 its")
_alg1.LOOP_MAX_MEMBERS = 64
for rep in range(3):
    t0 = time.perf_counter()
    sol = solver_single.solve_single(prob, solver_single.SingleParams())
    dt = time.perf_counter() - t0
print(f"converged solve (API): {dt * 1e3:.2f} ms, {sol.iterations} its, converged={sol.converged}")
for rep in range(3):
    t0 = time.perf_counter()
    sol = solver_single.solve_single(prob, solver_single.SingleParams(max_iter=100, tol=0.0))
    dt = time.perf_counter() - t0
print(f"100-it solve (API): {dt * 1e3:.2f} ms")
