"""Device time of the stable top-k (tro_topk_stable_f64) at the C4 shapes (CUDA events)."""
import json
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2408_10731_b200.solver_priest import _topk  # noqa: E402

for n, k in ((16384, 8192), (16384, 256), (131072, 65536), (131072, 256), (1048576, 8192)):
    keys = torch.as_tensor(np.random.default_rng(0).normal(size=n), device="cuda")
    for _ in range(3):
        _topk(keys, k)
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(20):
        _topk(keys, k)
    b.record()
    torch.cuda.synchronize()
    print(json.dumps({"n": n, "k": k, "us": round(a.elapsed_time(b) / 20 * 1e3, 1)}))
