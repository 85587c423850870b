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
