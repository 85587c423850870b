"""Measure the B200's fp64 FMA throughput (the roofline denominator of the FP-bound PRIEST projection)."""
import ctypes
import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2408_10731_b200 import _lib  # noqa: E402

lib = _lib.load()
scratch = torch.zeros(256, dtype=torch.float64, device="cuda")
blocks = torch.cuda.get_device_properties(0).multi_processor_count * 8
iters = 20000
for _ in range(2):
    _lib.check(lib.tro_fp64_fma_probe(iters, blocks, scratch.data_ptr(), ctypes.c_void_p(_lib.stream_handle())), "probe")
torch.cuda.synchronize()
best = 0.0
for _ in range(5):
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    _lib.check(lib.tro_fp64_fma_probe(iters, blocks, scratch.data_ptr(), ctypes.c_void_p(_lib.stream_handle())), "probe")
    b.record()
    torch.cuda.synchronize()
    s = a.elapsed_time(b) / 1e3
    best = max(best, blocks * 256 * iters * 8 * 2 / s / 1e12)
out = {"fp64_fma_tflops": best, "how": f"{blocks} blocks x 256 threads x {iters} x 8 independent DFMA chains, best of 5"}
print(json.dumps(out))
