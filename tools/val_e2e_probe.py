"""Where does the validation e2e time go (pinned coefficients in, results out)?"""
import os, sys, time
sys.path.insert(0, os.getcwd())
import numpy as np, torch
import bench
from paper_2408_10731_b200 import metrics as MT

basis, sc, xi_all = bench.val_inputs(131072)
t = basis.grid.timestamps
xi_pin = torch.as_tensor(xi_all).pin_memory()
xi_dev = xi_pin.cuda()


def tm(label, f, n=10):
    for _ in range(3):
        f()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(n):
        f()
    torch.cuda.synchronize()
    print(f"{label:40s} {(time.perf_counter() - t0) / n * 1e3:8.3f} ms", flush=True)


tm("device in, device out", lambda: MT.validate_batch(sc, t, xi=xi_dev, basis=basis, return_device=True))
tm("device in, host out", lambda: MT.validate_batch(sc, t, xi=xi_dev, basis=basis))
tm("h2d only (pinned, 34.6 MB)", lambda: xi_pin.to("cuda", non_blocking=True))
out = torch.empty((131072, 5), dtype=torch.float64, device="cuda")
tm("d2h pageable (5.2 MB)", lambda: out.cpu())
hp = torch.empty((131072, 5), dtype=torch.float64, pin_memory=True)
tm("d2h pinned (5.2 MB)", lambda: hp.copy_(out, non_blocking=True))
tm("pinned alloc 5.2 MB", lambda: torch.empty((131072, 5), dtype=torch.float64, pin_memory=True))
for k in (1, 2, 4, 8):
    MT._PIPE_MAX_CHUNKS = k
    MT._PIPE_MIN_CHUNK = 131072 // k
    tm(f"pinned in, host out, chunks {k}", lambda: MT.validate_batch(sc, t, xi=xi_pin, basis=basis))
