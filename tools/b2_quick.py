"""Quick Alg. 2 timing on the C2-alt recipe (N_b 1024, n_o 50, 200 iterations)."""
import os
import sys
import time

sys.path.insert(0, os.path.join(os.path.dirname(os.path.abspath(__file__)), ".."))

import torch

from paper_2408_10731_b200 import scenarios
from paper_2408_10731_b200 import solver_batch as SB

NB = int(os.environ.get("B2_NB", "1024"))
prob = scenarios.batch2d_problem(n_o=50, n_batch=NB)
params = SB.BatchParams(max_iter=200)
for rep in range(int(os.environ.get("B2_REPS", "3"))):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    r = SB.solve_batch_opt(prob, params, seed=0)
    torch.cuda.synchronize()
    dt = time.perf_counter() - t0
    print(f"rep {rep}: {dt * 1e3:.1f} ms/solve  {NB * 200 / dt:.3e} traj-it/s  best={r.best_index} "
          f"feasible={int(r.feasible.sum())} rho={r.state.rho:.3f}")
# device-only timing of the iteration loop
struct = SB._Structure(prob)
st = SB.init_state(prob, SB._default_samples(prob, struct.m, None, None, 0), params)
eng, lv, given = SB._engine_for(st, prob, struct, params, max_hist=400)
eng.prime(given)
eng.run(25)
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
eng.run(200)
e1.record()
torch.cuda.synchronize()
ms = e0.elapsed_time(e1)
print(f"device loop: {ms:.3f} ms / 200 it = {ms / 200 * 1e3:.1f} us/it, {NB * 200 / ms * 1e3:.3e} traj-it/s")
