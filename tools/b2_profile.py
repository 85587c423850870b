"""Alg. 2 C2-alt device loop for profiling: prime + N iterations (no host timing)."""
import os
import sys

sys.path.insert(0, os.path.join(os.path.dirname(os.path.abspath(__file__)), ".."))
import torch  # noqa: E402

from paper_2408_10731_b200 import scenarios  # noqa: E402
from paper_2408_10731_b200 import solver_batch as SB  # noqa: E402

n_o = int(os.environ.get("B2_NO", "50"))
n_b = int(os.environ.get("B2_NB", "1024"))
iters = int(os.environ.get("B2_IT", "60"))
prob = scenarios.batch2d_problem(n_o=n_o, n_batch=n_b)
params = SB.BatchParams(max_iter=iters)
struct = SB._Structure(prob)
st = SB.init_state(prob, SB._default_samples(prob, struct.m, None, None, 0), params)
eng, lv, given = SB._engine_for(st, prob, struct, params, max_hist=iters)
eng.prime(given)
for _ in range(iters):
    eng.iterate()
torch.cuda.synchronize()
print("done", eng.ints_host())
