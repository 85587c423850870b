"""C1 e2e breakdown: solve_single's phases (perf_counter, synchronized)."""
import os, sys, time
sys.path.insert(0, os.getcwd())
import numpy as np, torch
from paper_2408_10731_b200 import scenarios, solver_single as S

prob = scenarios.c1_problem()
prm = S.SingleParams(max_iter=100, tol=0.0)
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
    torch.cuda.synchronize(); a = time.perf_counter(); r = f(); torch.cuda.synchronize()
    acc[name] = acc.get(name, 0) + time.perf_counter() - a
    return r
for _ in range(N):
    eng = ph("engine", lambda: S._cached_engine(prob, prm, max_hist=100))
    ph("reset+init", lambda: (eng.reset_cold(), eng.cold_init()))
    ph("run", lambda: eng.run(100, use_graph=True, chunk=25, check_every=50))
    ph("raise_if_failed", lambda: S._raise_if_failed(eng))
    st = S.SingleState(xi=None, d=None, alpha=None, beta=None, cos_a=None, sin_a=None, cos_b=None, sin_b=None,
                       lam_pos=None, lam_cos_a=None, lam_sin_a=None, lam_cos_b=None, lam_sin_b=None, rho=1.0, rho_o=1.0)
    ph("download", lambda: S._download(eng, into=st))
    ph("hist", lambda: eng.hist[0, :int(eng.n_hist[0].item())].cpu().numpy())
for k, v in acc.items():
    print(f"{k:16s} {v / N * 1e3:.3f} ms")
