"""C1 in-kernel loop time (100 fixed iterations, half layout, the bench's engine) for the current library."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2408_10731_b200 import scenarios, solver_single  # noqa: E402
from paper_2408_10731_b200.solver_single import SingleBatch, make_batch_engine  # noqa: E402

prob = scenarios.c1_problem()
eng = make_batch_engine(SingleBatch.from_problems([prob]), solver_single.SingleParams(max_iter=100, tol=0.0),
                        layout="half")
best = 1e9
for _ in range(5):
    eng.reset_cold()
    eng.cold_init()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    eng.run(100, loop=True)
    b.record()
    torch.cuda.synchronize()
    best = min(best, a.elapsed_time(b))
print(f"{os.environ.get('TRO_LIB_PATH', 'default')}: {best:.3f} ms / 100 its")
