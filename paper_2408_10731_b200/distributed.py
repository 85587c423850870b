"""Member sharding across GPUs (one process per GPU, torch.distributed).

Batched Alg. 1 members are independent problems (per-member rho schedule,
convergence and history, solver_single.py:407-450), so a batch shards into
contiguous member ranges with NO per-iteration communication.
Each rank solves its range on its own GPU; the only collective is one
all-gather of per-shard summaries at the end of a solve (NCCL over
NVLink/NVSwitch on a B200 box, gloo in the CPU tests).
"""

from __future__ import annotations

import torch
import torch.distributed as dist


def shard_range(total: int, rank: int, world: int) -> tuple[int, int]:
    """Contiguous member range [lo, hi) of `rank`: member i lives on rank floor(i * world / total)."""
    if world < 1 or not 0 <= rank < world:
        raise ValueError("need 0 <= rank < world")
    return total * rank // world, total * (rank + 1) // world


def shard_summary(res_max: torch.Tensor, res_norm: torch.Tensor, converged: torch.Tensor, lo: int) -> torch.Tensor:
    """Per-shard summary: [best max|r|, its global member index, converged count, sum of norms, members].

    Exact quantities only (min / argmin / counts; the norm sum is informational), so the
    merged result does not depend on the number of shards."""
    n = res_max.numel()
    if n == 0:
        return torch.tensor([float("inf"), -1.0, 0.0, 0.0, 0.0], dtype=torch.float64, device=res_max.device)
    k = torch.argmin(res_max)  # first index on ties, like np.argmin
    return torch.stack([res_max[k].double(), (k + lo).double(), converged.sum().double(),
                        res_norm.double().sum(), torch.tensor(float(n), dtype=torch.float64, device=res_max.device)])


def merge_summaries(parts: list[torch.Tensor]) -> dict:
    """Global best member (smallest max|r|, first global index on ties) and totals."""
    best, best_idx = float("inf"), -1
    conv, members = 0, 0
    for p in parts:
        v = p.double().cpu().tolist()
        if v[0] < best or (v[0] == best and 0 <= v[1] < best_idx):
            best, best_idx = v[0], int(v[1])
        conv += int(v[2])
        members += int(v[4])
    return {"best_residual_max": best, "best_member": best_idx, "converged": conv, "members": members}


def gather_summaries(summary: torch.Tensor) -> dict:
    """All-gather the per-shard summaries (one tiny collective per solve) and merge them."""
    if not dist.is_available() or not dist.is_initialized() or dist.get_world_size() == 1:
        return merge_summaries([summary])
    out = [torch.empty_like(summary) for _ in range(dist.get_world_size())]
    dist.all_gather(out, summary)
    return merge_summaries(out)
