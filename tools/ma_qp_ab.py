"""Same-box timing of the multi-agent QP step at C3 (4096 problems x 16 agents): DMMA (tro_ma_run mode 3)
vs the Ozaki int8 tensor-core GEMM (tro_ma_qp_ozaki), CUDA events over repeated launches."""
import json
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests"))
from test_ozaki_gpu import _c3  # noqa: E402

from paper_2408_10731_b200 import solver_multiagent as MA  # noqa: E402


def main():
    n = int(sys.argv[1]) if len(sys.argv) > 1 else 4096
    reps = 20
    params = MA.JointParams(max_iter=200, rho_final=1e3)
    probs = _c3(n)
    struct = MA._Structure(probs[0], params)
    b_eq = np.stack([MA._b_eq(p) for p in probs])
    for qp, sl in (("dmma", 0), ("ozaki", 8), ("ozaki", 7), ("ozaki", 6)):
        e = MA.MaEngine(struct, b_eq, None, params, qp=qp, ozaki_slices=sl or 8)
        e.reset()
        e.init()
        e.run(3, use_graph=False, check_every=0)
        fn = (lambda: e._call(3)) if qp == "dmma" else e.qp_ozaki
        for _ in range(3):
            fn()
        torch.cuda.synchronize()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        for _ in range(reps):
            fn()
        b.record()
        torch.cuda.synchronize()
        us = a.elapsed_time(b) / reps * 1e3
        nv, nk = struct.n_a * struct.m, e.kinv.shape[1]
        flops = 2.0 * nv * nk * 3 * n
        print(json.dumps({"qp": qp, "slices": sl, "problems": n, "us_per_launch": round(us, 2),
                          "fp64_equiv_TFLOPs": round(flops / us / 1e6, 2)}), flush=True)
        del e
        torch.cuda.empty_cache()


if __name__ == "__main__":
    main()
