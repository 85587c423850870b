"""Multi-rank member sharding on CPU (gloo, world_size 2): the path the NCCL run takes."""

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2408_10731_b200.distributed import gather_summaries, merge_summaries, shard_range, shard_summary


def test_shard_range_partitions_exactly():
    for total in (1, 7, 1024, 131072):
        for world in (1, 2, 3, 4, 8):
            if world > total:
                continue
            ranges = [shard_range(total, r, world) for r in range(world)]
            assert ranges[0][0] == 0 and ranges[-1][1] == total
            assert all(a[1] == b[0] for a, b in zip(ranges, ranges[1:]))
            sizes = [hi - lo for lo, hi in ranges]
            assert max(sizes) - min(sizes) <= 1
    with pytest.raises(ValueError):
        shard_range(10, 2, 2)


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, res_max, res_norm, conv, out_q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    lo, hi = shard_range(len(res_max), rank, world)
    summ = shard_summary(torch.tensor(res_max[lo:hi]), torch.tensor(res_norm[lo:hi]),
                         torch.tensor(conv[lo:hi]), lo)
    merged = gather_summaries(summ)
    out_q.put((rank, merged))
    dist.destroy_process_group()


def test_two_rank_gather_matches_single_rank():
    rng = np.random.default_rng(0)
    n = 37
    res_max = np.round(rng.uniform(0, 1, n), 2)  # ties across the shard boundary
    res_max[[3, 30]] = res_max.min() - 0.5
    res_norm = rng.uniform(0, 5, n)
    conv = res_max <= 0.2
    single = merge_summaries([shard_summary(torch.tensor(res_max), torch.tensor(res_norm), torch.tensor(conv), 0)])
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, res_max, res_norm, conv, q)) for r in range(2)]
    for p in procs:
        p.start()
    got = [q.get(timeout=120) for _ in procs]
    for p in procs:
        p.join(timeout=60)
    for _, merged in got:
        assert merged == single
    assert single["best_member"] == 3 and single["members"] == n and single["converged"] == int(conv.sum())


# ------------------------------------------------------------------ Alg. 2: batch-global rho across ranks
def _b2_truth(res_norm, res_max):
    nan = np.isnan(res_norm)
    k = int(np.argmax(nan)) if nan.any() else int(np.argmin(res_norm))
    return res_norm[k], k, res_max[k], np.min(res_max)


def _b2_worker(rank, world, port, res_norm, res_max, aug, feas, out_q):
    from paper_2408_10731_b200.distributed import b2_global_best, b2_local_summary, b2_merge

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    lo, hi = shard_range(len(res_norm), rank, world)
    mine = torch.tensor(b2_local_summary(res_norm[lo:hi], res_max[lo:hi], lo))
    parts = [torch.empty(4, dtype=torch.float64) for _ in range(world)]
    dist.all_gather(parts, mine)
    merged = b2_merge(torch.stack(parts).numpy())
    best = b2_global_best(aug[lo:hi], feas[lo:hi], lo)
    out_q.put((rank, merged, best))
    dist.destroy_process_group()


@pytest.mark.parametrize("case", ["ties", "nan"])
def test_alg2_shard_summaries_merge_to_the_batch_decision(case):
    """Two gloo ranks: the per-iteration shard summaries of a sharded Alg. 2 batch, all-gathered and merged
    in rank order, give the single-batch argmin / min (solver_batch.py:454-460) and the final ranking."""
    rng = np.random.default_rng(1)
    n = 41
    res_norm = np.round(rng.uniform(0, 1, n), 2)
    res_norm[[7, 33]] = res_norm.min() - 0.25  # tie across the shard boundary: first index wins
    res_max = rng.uniform(0, 1, n)
    if case == "nan":
        res_norm[[25, 30]] = np.nan  # numpy's argmin returns the first NaN
        res_max[12] = np.nan
    aug = np.round(rng.uniform(0, 3, n), 1)
    feas = rng.uniform(0, 1, n) < 0.6
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_b2_worker, args=(r, 2, port, res_norm, res_max, aug, feas, q)) for r in range(2)]
    for p in procs:
        p.start()
    got = [q.get(timeout=120) for _ in range(2)]
    for p in procs:
        p.join(timeout=60)
    b, k, bm, mm = _b2_truth(res_norm, res_max)
    full = np.where(feas, aug, np.inf)
    for _, (mb, mk, mbm, mmm), best in got:
        assert mk == k
        assert (np.isnan(b) and np.isnan(mb)) or mb == b
        assert mbm == bm or (np.isnan(bm) and np.isnan(mbm))
        assert (np.isnan(mm) and np.isnan(mmm)) or mmm == mm
        assert best == int(np.argmin(full))


# ------------------------------------------------------------------ PRIEST: candidate all-gather == global stable top-k
def _topk_worker(rank, world, port, scores, k, out_q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    lo, hi = shard_range(len(scores), rank, world)
    local = scores[lo:hi]
    cand = np.argsort(local, kind="stable")[:min(k, hi - lo)]
    mine = torch.tensor(np.stack([local[cand], cand + lo], axis=1))
    parts = [torch.empty_like(mine) for _ in range(world)]
    dist.all_gather(parts, mine)
    rows = torch.cat(parts).numpy()
    keep = np.argsort(rows[:, 0], kind="stable")[:k]
    out_q.put((rank, rows[keep, 1].astype(np.int64)))
    dist.destroy_process_group()


@pytest.mark.parametrize("k", [5, 30])
def test_priest_candidate_gather_is_the_global_stable_topk(k):
    """ShardedRound's merge on two gloo ranks: local stable top-k, rank-ordered all-gather, stable top-k
    of the gathered scores == np.argsort(all scores, kind='stable')[:k] (ties across the boundary)."""
    rng = np.random.default_rng(2)
    scores = np.round(rng.uniform(0, 1, 40), 1)  # many ties, across the shard boundary
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_topk_worker, args=(r, 2, port, scores, k, q)) for r in range(2)]
    for p in procs:
        p.start()
    got = [q.get(timeout=120) for _ in range(2)]
    for p in procs:
        p.join(timeout=60)
    for _, idx in got:
        np.testing.assert_array_equal(idx, np.argsort(scores, kind="stable")[:k])


# ------------------------------------------------------------------ Alg. 1: sharded public entry point
class _FakeSol:
    """Stands in for a BatchSolution in the host-logic test (deterministic per-member values)."""

    def __init__(self, sub):
        from paper_2408_10731_b200.solver_single import BatchResult

        bv = np.asarray(sub.bvals)
        B = bv.shape[0]
        xi = np.repeat(bv[:, :, :1], 11, axis=2) * np.arange(11)[None, None, :]
        rmax = np.round(np.abs(bv[:, 1, 0]) + np.abs(bv[:, 2, 3]), 1)
        self._r = BatchResult(xi=xi, residual_norm=2 * rmax, residual_max=rmax, rho_o=np.ones(B),
                              converged=rmax <= 0.5, iterations=np.full(B, 7), n_factorizations=np.ones(B, int),
                              history=None)
        self.residual_max = torch.as_tensor(rmax)

    def numpy(self):
        return self._r


def _fake_solve(sub, params=None, **kw):
    return _FakeSol(sub)


def _sharded_worker(rank, world, port, out_q):
    from paper_2408_10731_b200 import scenarios
    from paper_2408_10731_b200.basis import build_basis
    from paper_2408_10731_b200.distributed import solve_single_batch_sharded

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    batch = scenarios.flow3d_batch(5, range(23), basis=build_basis(0.0, 10.0, 100, 10))
    local, merged, full = solve_single_batch_sharded(batch, None, gather_results=True, solve=_fake_solve)
    out_q.put((rank, local.xi.shape[0], merged, {k: v.tolist() for k, v in full.items()}))
    dist.destroy_process_group()


def test_alg1_sharded_entry_point_two_ranks_gloo():
    from paper_2408_10731_b200 import scenarios
    from paper_2408_10731_b200.basis import build_basis
    from paper_2408_10731_b200.distributed import solve_single_batch_sharded

    batch = scenarios.flow3d_batch(5, range(23), basis=build_basis(0.0, 10.0, 100, 10))
    _, single, full1 = solve_single_batch_sharded(batch, None, gather_results=True, solve=_fake_solve)
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_sharded_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    got = sorted([q.get(timeout=180) for _ in procs])
    for p in procs:
        p.join(timeout=60)
    assert [g[1] for g in got] == [11, 12]  # contiguous ranges [0, 11) and [11, 23)
    for _, _, merged, full in got:
        assert merged == single
        for k, v in full1.items():
            np.testing.assert_array_equal(np.asarray(full[k]), v)
