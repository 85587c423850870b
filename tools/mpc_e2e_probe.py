"""MPC e2e: fleet construction vs episode vs results (perf_counter, synchronized) + cProfile of one e2e step."""
import cProfile, os, pstats, sys, time
sys.path.insert(0, os.getcwd())
import torch
import bench
from paper_2408_10731_b200.mpc import MpcFleet

sc, starts, goals = bench.mpc_inputs(1024)
f = MpcFleet(sc, starts, goals, step_budget=40, layout="half")
f.run(30, early_exit=False)
torch.cuda.synchronize()
for _ in range(2):
    t0 = time.perf_counter(); f2 = MpcFleet(sc, starts, goals, step_budget=40, layout="half"); torch.cuda.synchronize()
    t1 = time.perf_counter(); fr = f2.run(30, early_exit=False); torch.cuda.synchronize(); t2 = time.perf_counter()
    t3 = time.perf_counter(); fr = f.run(30, early_exit=False); torch.cuda.synchronize(); t4 = time.perf_counter()
    print(f"construct {1e3*(t1-t0):.1f} ms  run(new fleet) {1e3*(t2-t1):.1f} ms  run(reused fleet) {1e3*(t4-t3):.1f} ms")
pr = cProfile.Profile(); pr.enable()
MpcFleet(sc, starts, goals, step_budget=40, layout="half").run(30, early_exit=False)
torch.cuda.synchronize(); pr.disable()
pstats.Stats(pr).sort_stats("tottime").print_stats(15)
