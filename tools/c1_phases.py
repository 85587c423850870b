"""Per-phase cycle counts of the C1 in-kernel loop (diagnostic library built with -DTRO_PHASE_PROF):
    TRO_LIB_PATH=paper_2408_10731_b200/csrc/build/variants/libtrajopt_b200_phase.so python tools/c1_phases.py"""
import ctypes
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2408_10731_b200 import _lib, scenarios, solver_single  # noqa: E402

prob = scenarios.c1_problem()
for _ in range(3):
    sol = solver_single.solve_single(prob, solver_single.SingleParams())
torch.cuda.synchronize()
lib = _lib.load()
buf = (ctypes.c_longlong * 8192)()
lib.tro_debug_phase(buf, 8192)
a = np.frombuffer(buf, dtype=np.int64).reshape(1024, 8)[:sol.iterations - 1]
d = np.diff(np.concatenate([np.zeros((a.shape[0], 1), dtype=np.int64), a[:, 1:7]], axis=1), axis=1)
names = ["stage", "q_lin", "K^-1 apply", "positions", "elements + partials", "sums + schedule"]
med = np.median(d, axis=0)
print("median cycles per phase:", dict(zip(names, med.tolist())), "total", float(med.sum()))
print("iteration cycles (loop top to loop top, median):", float(np.median(np.diff(a[:, 6]))) if False else "")
