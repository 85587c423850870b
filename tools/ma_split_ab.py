"""C3 element-kernel A/B across library builds (TRO_LIB_PATH): ms per iteration + the state after 25
iterations, saved for a bitwise comparison between builds.  usage: python tools/ma_split_ab.py OUT.npz"""
import os, sys
sys.path.insert(0, os.getcwd())
import numpy as np, torch
import bench
from paper_2408_10731_b200 import solver_multiagent as MA
probs = bench.c3_problems(0, 4096)
params = MA.JointParams(max_iter=200, rho_final=1e3, tol_norm=0.0)
struct = MA._Structure(probs[0], params)
beq = np.stack([MA._b_eq(p) for p in probs])
eng = MA.MaEngine(struct, beq, None, params, split_qp=True)
eng.init()
for _ in range(5):
    eng.iterate()
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(20):
    eng.iterate()
e1.record()
torch.cuda.synchronize()
ms = e0.elapsed_time(e1) / 20
print(os.environ.get("TRO_LIB_PATH", "base"), "ms/iter", round(ms, 4))
np.savez(sys.argv[1], xi=eng.xi.cpu().numpy(), ms=ms)
