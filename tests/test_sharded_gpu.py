"""The real sharded Alg. 1 solve (distributed.solve_single_batch_sharded) as two processes on one GPU.

Members are independent, so the sharded path has no per-iteration collective; the two
ranks only meet in the final summary all-gather (gloo here: both ranks share the one GPU this suite runs
on, and their kernels never wait on each other).  The gathered per-member results must equal the
single-process solve of the whole batch bit for bit, and the merged summary must equal the one-shard one.
"""

import os
import socket

import numpy as np
import pytest
import torch.multiprocessing as mp

pytestmark = pytest.mark.gpu

N_MEMBERS = 140  # > LOOP_MAX_MEMBERS per shard (TMA kernel + graph); <= one CTA per SM: no tail split anywhere


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _batch():
    from paper_2408_10731_b200 import scenarios
    from paper_2408_10731_b200.basis import build_basis

    return scenarios.flow3d_batch(50, range(N_MEMBERS), basis=build_basis(0.0, 10.0, 100, 10))


def _params():
    from paper_2408_10731_b200.solver_single import SingleParams

    return SingleParams(max_iter=60, tol=1e-3)


def _worker(rank, world, port, q):
    import torch
    import torch.distributed as dist

    from paper_2408_10731_b200.distributed import solve_single_batch_sharded

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    torch.cuda.set_device(0)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        _, merged, full = solve_single_batch_sharded(_batch(), _params(), gather_results=True, layout="half")
        q.put((rank, merged, {k: np.asarray(v) for k, v in full.items()}, None))
    except Exception as exc:  # noqa: BLE001 - report to the parent
        q.put((rank, None, None, repr(exc)))
    finally:
        dist.destroy_process_group()


def test_two_rank_sharded_solve_equals_single_process():
    from paper_2408_10731_b200.distributed import solve_single_batch_sharded

    _, single, full1 = solve_single_batch_sharded(_batch(), _params(), gather_results=True, layout="half")
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    got = [q.get(timeout=600) for _ in procs]
    for p in procs:
        p.join(timeout=120)
    for rank, merged, full, err in got:
        assert err is None, err
        assert merged == single
        for k, v in full1.items():
            np.testing.assert_array_equal(full[k], v, err_msg=k)
    assert single["members"] == N_MEMBERS


# ------------------------------------------------------------------ multi-agent (Alg. 5) shards
N_PROBLEMS = 24


def _ma_problems():
    from paper_2408_10731_b200 import solver_multiagent as MA
    from paper_2408_10731_b200.basis import AxisBoundary, build_basis
    from paper_2408_10731_b200.geometry import EllipsoidShape

    b = build_basis(0.0, 10.0, 100, 10)
    out = []
    for s in range(N_PROBLEMS):
        rng = np.random.default_rng(100 + s)
        starts, goals = rng.uniform(-3.0, 3.0, (8, 3)), rng.uniform(-3.0, 3.0, (8, 3))
        bnds = [tuple(AxisBoundary(p0=float(starts[i, k]), p1=float(goals[i, k])) for k in range(3))
                for i in range(8)]
        out.append(MA.MultiAgentProblem(basis=b, boundaries=bnds, agent_shape=EllipsoidShape(0.3, 0.45)))
    return out


def _ma_params():
    from paper_2408_10731_b200 import solver_multiagent as MA

    return MA.JointParams(max_iter=30, rho_final=1e3)


def _ma_worker(rank, world, port, q):
    import torch
    import torch.distributed as dist

    from paper_2408_10731_b200.distributed import solve_joint_batch_sharded

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    torch.cuda.set_device(0)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        _, merged, full = solve_joint_batch_sharded(_ma_problems(), _ma_params(), gather_results=True)
        q.put((rank, merged, full, None))
    except Exception as exc:  # noqa: BLE001 - report to the parent
        q.put((rank, None, None, repr(exc)))
    finally:
        dist.destroy_process_group()


def test_two_rank_sharded_joint_solve_equals_single_process():
    """solve_joint_batch_sharded: two ranks (one GPU, gloo) reproduce the one-process batch bit for bit."""
    from paper_2408_10731_b200.distributed import solve_joint_batch_sharded

    _, single, full1 = solve_joint_batch_sharded(_ma_problems(), _ma_params(), gather_results=True)
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_ma_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    got = [q.get(timeout=600) for _ in procs]
    for p in procs:
        p.join(timeout=120)
    for rank, merged, full, err in got:
        assert err is None, err
        assert merged == single
        for k, v in full1.items():
            np.testing.assert_array_equal(full[k], v, err_msg=k)
    assert single["members"] == N_PROBLEMS
