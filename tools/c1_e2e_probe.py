"""C1 e2e breakdown: solve_single's phases (perf_counter, synchronized) for the converged solve."""
import os
import sys
import time

sys.path.insert(0, os.getcwd())
import torch  # noqa: E402

from paper_2408_10731_b200 import scenarios  # noqa: E402
from paper_2408_10731_b200 import solver_single as S  # noqa: E402

prob = scenarios.c1_problem()
prm = S.SingleParams()
for _ in range(3):
    S.solve_single(prob, prm)
torch.cuda.synchronize()
N = 30
t0 = time.perf_counter()
for _ in range(N):
    S.solve_single(prob, prm)
torch.cuda.synchronize()
print("solve_single", (time.perf_counter() - t0) / N * 1e3, "ms")
acc = {}


def ph(name, f):
    torch.cuda.synchronize()
    a = time.perf_counter()
    r = f()
    torch.cuda.synchronize()
    acc[name] = acc.get(name, 0) + time.perf_counter() - a
    return r


for _ in range(N):
    eng = ph("engine lookup", lambda: S._cached_engine(prob, prm, max_hist=prm.max_iter))
    ph("cold init", lambda: eng.cold_init())
    ph("run", lambda: eng.run(prm.max_iter, use_graph=True, chunk=25, check_every=50))
    snap = ph("snapshot", lambda: S._snapshot(eng))
    st = S.SingleState(xi=None, d=None, alpha=None, beta=None, cos_a=None, sin_a=None, cos_b=None, sin_b=None,
                       lam_pos=None, lam_cos_a=None, lam_sin_a=None, lam_cos_b=None, lam_sin_b=None, rho=1.0, rho_o=1.0)
    ph("download", lambda: S._download(eng, into=st, snap=snap))
for k, v in acc.items():
    print(f"{k:16s} {v / N * 1e3:.3f} ms")
