"""Launch-geometry / variant sweep for the fused Alg. 1 kernel (device time, CUDA events).

    TRO_LIB_PATH=paper_2408_10731_b200/csrc/build/variants/libtrajopt_b200_u1.so \
        python tools/tune_alg1.py --members 16384 --n-obs 100 --groups 2,4,5 --dtype f64
"""
import argparse
import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2408_10731_b200 import scenarios  # noqa: E402
from paper_2408_10731_b200.basis import build_basis  # noqa: E402
from paper_2408_10731_b200.solver_single import SingleParams, make_batch_engine  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--members", type=int, default=16384)
    ap.add_argument("--n-obs", type=int, default=100)
    ap.add_argument("--groups", default="0")
    ap.add_argument("--dtype", default="f64")
    ap.add_argument("--iters", type=int, default=30)
    ap.add_argument("--tag", default=os.path.basename(os.environ.get("TRO_LIB_PATH", "default")))
    ap.add_argument("--no-tma", action="store_true")
    ap.add_argument("--layout", default="angle")
    ap.add_argument("--no-lin", action="store_true", help="stream the track rows (no register-generated tracks)")
    a = ap.parse_args()
    dtype = torch.float64 if a.dtype == "f64" else torch.float32
    s = 8 if a.dtype == "f64" else 4
    basis = build_basis(0.0, 10.0, 100, 10)
    batch = scenarios.flow3d_batch(a.n_obs, range(a.members), basis=basis)
    params = SingleParams(max_iter=a.iters, tol=0.0)
    peak = json.load(open("MEASURED_PEAKS.json"))["hbm_gbs"] if os.path.exists("MEASURED_PEAKS.json") else 6650.0
    for G in [int(x) for x in a.groups.split(",")]:
        eng = make_batch_engine(batch, params, dtype=dtype, groups=G, layout=a.layout)
        if a.no_tma:
            eng.base_flags = 2
        if a.no_lin:
            eng._consts.track_lin = None
        eng.cold_init()
        eng.run(5, use_graph=False)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(a.iters):
            eng.iterate(2)
        e1.record()
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1) / a.iters
        gbs = 2 * 9 * a.n_obs * 100 * s * a.members / (ms / 1e3) / 1e9
        print(json.dumps({"tag": a.tag + ("" if not a.no_tma else "+notma") + ("+nolin" if a.no_lin else "") + "+" + a.layout, "G": G, "ms_per_iter": round(ms, 4), "GBps": round(gbs, 1),
                          "frac": round(gbs / peak, 3), "dtype": a.dtype, "members": a.members, "n_obs": a.n_obs}))
        del eng
        torch.cuda.empty_cache()


if __name__ == "__main__":
    main()
