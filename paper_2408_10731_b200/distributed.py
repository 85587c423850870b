"""Member sharding across GPUs (one process per GPU, torch.distributed).

Batched Alg. 1 members are independent problems (per-member rho schedule,
convergence and history, solver_single.py:407-450), so a batch shards into
contiguous member ranges with NO per-iteration communication.
Each rank solves its range on its own GPU; the only collective is one
all-gather of per-shard summaries at the end of a solve (NCCL over
NVLink/NVSwitch on a B200 box, gloo in the CPU tests).
"""

from __future__ import annotations

import numpy as np
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


def gather_summaries(summary: torch.Tensor, group=None) -> dict:
    """All-gather the per-shard summaries (one tiny collective per solve) and merge them.  NCCL gathers the
    device tensor; gloo (CPU tests, or ranks sharing one GPU) gathers a host copy."""
    if not dist.is_available() or not dist.is_initialized() or dist.get_world_size(group) == 1:
        return merge_summaries([summary])
    if dist.get_backend(group) != "nccl":
        summary = summary.cpu()
    out = [torch.empty_like(summary) for _ in range(dist.get_world_size(group))]
    dist.all_gather(out, summary, group=group)
    return merge_summaries(out)


def _world(group=None) -> tuple[int, int]:
    if dist.is_available() and dist.is_initialized():
        return dist.get_rank(group), dist.get_world_size(group)
    return 0, 1


def shard_batch(batch, rank: int, world: int):
    """This rank's contiguous member range of a solver_single.SingleBatch (shared basis and obstacles)."""
    from .solver_single import SingleBatch

    lo, hi = shard_range(batch.B, rank, world)
    des = None if batch.desired is None else np.asarray(batch.desired)[lo:hi]
    return lo, hi, SingleBatch(batch.basis, np.asarray(batch.bvals)[lo:hi], list(batch.obstacles), des,
                               batch.w_smooth, batch.w_track)


def solve_single_batch_sharded(batch, params=None, *, group=None, gather_results: bool = False, solve=None, **kw):
    """solve_single_batch over all ranks of `group` (one process per GPU): rank r solves members
    [shard_range(B, r, world)) with NO per-iteration communication (members are independent,
    solver_single.py:407-450), then ONE all-gather of the per-shard summaries.

    Returns (local BatchResult, merged summary, full results or None).  gather_results=True also
    all-gathers every rank's per-member results (xi, residuals, counters) into member order, which the
    bitwise shard-vs-single tests use; `solve` substitutes the per-shard solve (host-logic tests)."""
    from .solver_single import solve_single_batch

    rank, world = _world(group)
    if batch.B < world:
        raise ValueError("fewer members than ranks")
    lo, hi, sub = shard_batch(batch, rank, world)
    sol = (solve or solve_single_batch)(sub, params, **kw)
    local = sol.numpy()
    dev = sol.residual_max.device
    summary = shard_summary(torch.as_tensor(local.residual_max, device=dev),
                            torch.as_tensor(local.residual_norm, device=dev),
                            torch.as_tensor(local.converged, device=dev), lo)
    merged = gather_summaries(summary, group)
    full = None
    if gather_results:
        parts = [None] * world
        if world > 1:
            dist.all_gather_object(parts, local, group=group)
        else:
            parts = [local]
        full = {k: np.concatenate([getattr(p, k) for p in parts])
                for k in ("xi", "residual_norm", "residual_max", "rho_o", "converged", "iterations",
                          "n_factorizations")}
    return local, merged, full


def solve_joint_batch_sharded(problems: list, params=None, *, group=None, gather_results: bool = False, **kw):
    """solver_multiagent.solve_joint_batch over all ranks of `group`: rank r solves problems
    [shard_range(B, r, world)) with no per-iteration communication (joint problems are independent,
    solver_multiagent.py:300-368), then one all-gather of the per-shard summaries (max|r|, ||r||,
    converged, in problem order).  gather_results=True also all-gathers xi, the residuals, the counters and
    the levels for the bitwise shard-vs-single tests.  Returns (local engine, merged summary, full or None)."""
    from . import _lib
    from .solver_multiagent import solve_joint_batch

    rank, world = _world(group)
    if len(problems) < world:
        raise ValueError("fewer problems than ranks")
    lo, hi = shard_range(len(problems), rank, world)
    eng = solve_joint_batch(list(problems[lo:hi]), params, **kw)
    conv = (eng.status & _lib.TRO_CONVERGED) != 0
    merged = gather_summaries(shard_summary(eng.res_max, eng.res_norm, conv, lo), group)
    full = None
    if gather_results:
        local = {"xi": eng.xi.cpu().numpy(), "res_norm": eng.res_norm.cpu().numpy(),
                 "res_max": eng.res_max.cpu().numpy(), "iteration": eng.iteration.cpu().numpy(),
                 "level": eng.level.cpu().numpy(), "converged": conv.cpu().numpy()}
        parts = [None] * world
        if world > 1:
            dist.all_gather_object(parts, local, group=group)
        else:
            parts = [local]
        full = {k: np.concatenate([q[k] for q in parts]) for k in local}
    return eng, merged, full


# ------------------------------------------------------------------ Alg. 2 (batch-global rho)
# solve_batch_opt's penalty rule is batch-global (solver_batch.py:454-461): each iteration needs the
# best member (argmin of ||r||, first index; numpy returns the first NaN) and min_i max|r_i| over the
# WHOLE batch.  Sharded, every rank's last CTA writes a 4-double summary (best norm, best global index,
# its max|r|, min max|r|) (TRO_B2_SHARD), the summaries are all-gathered (NCCL, 32 B per rank per
# iteration) and every rank merges them in rank order (tro_b2_run mode 6), so all ranks take the
# single-GPU decisions bit for bit.  The numpy functions below state the same merge for the CPU tests.
def b2_local_summary(res_norm, res_max, offset: int):
    """numpy mirror of the kernel's shard summary: [best norm, best global index, its max, min max]."""
    import numpy as np

    res_norm, res_max = np.asarray(res_norm, float), np.asarray(res_max, float)
    if res_norm.size == 0:
        return np.array([np.inf, -1.0, 0.0, np.inf])
    nan = np.isnan(res_norm)
    k = int(np.argmax(nan)) if nan.any() else int(np.argmin(res_norm))
    return np.array([res_norm[k], float(offset + k), res_max[k], np.min(res_max)])


def b2_merge(rows):
    """numpy mirror of mode 6: merge rank-ordered shard summaries -> (best, index, best_max, min_max)."""
    import numpy as np

    rows = np.asarray(rows, float)
    ok = rows[:, 1] >= 0
    cand = rows[ok]
    nan = np.isnan(cand[:, 0])
    if nan.any():
        c = cand[nan]
        j = int(np.argmin(c[:, 1]))
    else:
        c = cand
        j = int(np.lexsort((c[:, 1], c[:, 0]))[0])
    return float(c[j, 0]), int(c[j, 1]), float(c[j, 2]), float(np.min(rows[:, 3]))


def b2_global_best(local_aug, local_feasible, offset: int, group=None):
    """Global ranking (solver_batch.py:471): argmin of aug over feasible members of the whole batch, first
    global index on ties; one all-gather of (best aug, index) per solve."""
    import numpy as np

    aug = np.where(np.asarray(local_feasible, bool), np.asarray(local_aug, float), np.inf)
    if aug.size and np.isfinite(aug).any():
        k = int(np.argmin(aug))
        mine = torch.tensor([aug[k], float(offset + k)], dtype=torch.float64)
    else:
        mine = torch.tensor([np.inf, -1.0], dtype=torch.float64)
    if dist.is_available() and dist.is_initialized() and dist.get_world_size(group) > 1:
        dev = torch.device("cuda", torch.cuda.current_device()) if dist.get_backend(group) == "nccl" else "cpu"
        parts = [torch.empty(2, dtype=torch.float64, device=dev) for _ in range(dist.get_world_size(group))]
        dist.all_gather(parts, mine.to(dev), group=group)
        rows = np.stack([p.cpu().numpy() for p in parts])
    else:
        rows = mine.numpy()[None]
    rows = rows[rows[:, 1] >= 0]
    if rows.size == 0:
        return None
    return int(rows[np.lexsort((rows[:, 1], rows[:, 0]))[0], 1])


def solve_batch_opt_sharded(problem, params=None, *, samples=None, mean=None, covariance=None, seed=0, group=None,
                            use_graph=True):
    """solve_batch_opt over all ranks of `group`: every rank draws the same samples (same seed), keeps its
    contiguous member range, and the batch-global rho decisions are merged each iteration (see above).
    Returns this rank's RankedSolutions (local members, best_index = GLOBAL index or None)."""
    import numpy as np

    from . import solver_batch as SB

    params = params or SB.BatchParams()
    world = dist.get_world_size(group) if dist.is_available() and dist.is_initialized() else 1
    rank = dist.get_rank(group) if world > 1 else 0
    struct = SB._structure_for(problem)
    if samples is None:
        samples = SB._default_samples(problem, struct.m, mean, covariance, seed)
    samples = np.asarray(samples, float)
    if samples.shape[0] < world:
        raise ValueError("fewer members than ranks")
    lo, hi = shard_range(samples.shape[0], rank, world)
    state = SB.init_state(problem, samples[lo:hi], params)
    lv = SB._levels(struct, float(state.rho), float(state.rho_psi), params.rho_growth, params.rho_cap)
    eng = SB._Engine(struct, hi - lo, lv, params=params, max_hist=params.max_iter, member_offset=lo)
    eng.load(state, 0)
    gathered = torch.zeros((world, 4), dtype=torch.float64, device=eng.device)
    n_iter = int(params.max_iter)
    if n_iter > 0:
        SB._ensure_factors(state, lv, 0)
        eng.prime(False)
    for _ in range(n_iter):
        eng.iterate()
        if world > 1:
            dist.all_gather_into_tensor(gathered, eng.shard, group=group)
        else:
            gathered.copy_(eng.shard[None])
        eng.merge(gathered)
    eng.run_mode(3, eng.flags)
    got = eng.fetch(("ints", "hist", "rank", "xi", "xi_psi", "psi", "lam", "lam_psi"))
    n_hist = int(got["ints"][3])
    hist = got["hist"][:n_hist] if n_iter > 0 else np.zeros((0, 4))
    if n_iter > 0:
        for name in ("xi", "xi_psi", "psi", "lam", "lam_psi"):
            setattr(state, name, got[name])
        state.iteration += n_iter
        used = SB._rho_level(lv, float(hist[-1, 2]), lv.rho_psi[lv.rho.index(float(hist[-1, 2]))])
        for k in range(1, used + 1):
            SB._ensure_factors(state, lv, k)
        level = int(got["ints"][0])
        state.rho, state.rho_psi = lv.rho[level], lv.rho_psi[level]
        state._imply(struct)
    rank_arr = got["rank"]
    feasible = (rank_arr[:, 0] <= params.tol) & SB._feasible_from_rank(rank_arr, problem, params.d_margin,
                                                                      params.kin_margin)
    costs = rank_arr[:, 5].copy()
    aug = costs + state.rho * rank_arr[:, 1]
    best = b2_global_best(aug, feasible, lo, group)
    return SB.RankedSolutions(
        trajectories=SB._TrajectoryList(problem.basis, state.xi, state.psi, struct.m), costs=costs, aug_costs=aug,
        residual_max=rank_arr[:, 0].copy(), residual_norm=rank_arr[:, 1].copy(), feasible=feasible, best_index=best,
        best_history=[{"norm": float(h[0]), "max_abs": float(h[1]), "rho": float(h[2])} for h in hist],
        iterations=state.iteration, n_factorizations=state.n_factorizations, state=state)
