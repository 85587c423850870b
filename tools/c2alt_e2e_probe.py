"""C2-alt e2e: where solve_batch_opt's host time goes (cProfile around 5 calls, samples from the host)."""
import cProfile, os, pstats, sys, time
sys.path.insert(0, os.getcwd())
import torch
from paper_2408_10731_b200 import scenarios, solver_batch as SB

prob = scenarios.batch2d_problem(n_o=50, n_batch=1024)
params = SB.BatchParams(max_iter=200)
struct = SB._structure_for(prob)
samples = SB._default_samples(prob, struct.m, None, None, 0)
for _ in range(2):
    SB.solve_batch_opt(prob, params, samples=samples)
torch.cuda.synchronize()
t0 = time.perf_counter()
for _ in range(5):
    SB.solve_batch_opt(prob, params, samples=samples)
torch.cuda.synchronize()
print("solve_batch_opt", (time.perf_counter() - t0) / 5 * 1e3, "ms")
pr = cProfile.Profile()
pr.enable()
for _ in range(5):
    SB.solve_batch_opt(prob, params, samples=samples)
torch.cuda.synchronize()
pr.disable()
pstats.Stats(pr).sort_stats("tottime").print_stats(18)
