"""Benchmark: batched Alg. 1 AM/AL trajectory optimization (trajectory-iterations / s).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config c5|c2|c1] [--dtype f64|f32]
    python bench.py --impl reference ...      # reference CPU path (oracle port) on host cores
    torchrun --nproc-per-node N bench.py --gpus N   # one process per GPU, NCCL

A step = one full solve (cold init + max_iter fused AM iterations) of the
configuration's member batch; value = members x AM iterations / step time
(device time, CUDA events, max over ranks).  Members are sharded contiguously
across ranks with no data-path collective; one NCCL all-gather of per-shard
summaries closes each step.  The per-element state (C5: 94 GB fp64) is far
larger than L2, so no explicit L2 flush is needed between iterations.

e2e: the same solve through the public batched API with the step's member
inputs (boundary values + linear cost terms) copied from pinned host memory
and the results (xi, residual max/norm, converged) copied back, inside the
timed region.
"""

from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

CONFIGS = {
    # name: (n_obs, members, n_iter, description)
    "c5": (100, 131072, 200, "C5: 131072 traj x 100 dyn. ellipsoids x n_p 100, 200 AM its (3-D)"),
    "c2": (50, 1024, 200, "C2: 1024 traj x 50 dyn. ellipsoids x n_p 100, 200 AM its (3-D)"),
    "c1": (10, 1, 100, "C1: 1 quadrotor x 10 static ellipsoids x n_p 100, 100 AM its (3-D)"),
    "c4": (100, 16384, 30, "C4: PRIEST CEM, 16384 samples, 8192 constraint elites, top-256, 100 static "
                           "ellipsoids, n_p 100, 30 inner its, 10 rounds (3-D)"),
}
C4_ROUNDS, C4_NCE, C4_NEL = 10, 8192, 256
CONFIGS["c3"] = (16, 4096, 200, "C3: 4096 joint problems x 16 quadrotors (120 pairs, ellipsoid 0.3/0.45) x n_p 100, "
                                "200 iterations (rho_final 1e3, tol 0: fixed work)")
CONFIGS["c2alt"] = (50, 1024, 200, "C2-alt (Alg. 2): 1024 members x 50 dyn. circles (dynamic-flow, seed 0) x "
                                   "n_p 100, 1 footprint circle + heading, 200 batch iterations (2-D)")
CONFIGS["val"] = (100, 131072, 1, "Validation (SURVEY 8(f) row 3): 131072 C5 trajectories x 100 raw dynamic ellipsoids "
                                  "x n_p 100: smoothness, tracking, arc length, worst incursion, clearance bound")
CONFIGS["mpc"] = (50, 1024, 40, "MPC fleet (SURVEY 8(f) row 2): 1024 robots in the C2 field (50 dyn. ellipsoids, "
                                "n_p 100, 3-D), receding horizon: 30 control steps x 40 warm AM its, 10 samples "
                                "executed per step")
MPC_STEPS = 30
VAL_FLOPS_ELEM = 24  # per (member, obstacle, sample): predicted centre 6, offset 3, quad 8, sqrt 1, worst 2, clearance 2
B2_FLOPS_ELEM = 20  # per (circle, obstacle, sample): deltas, unit vector, num / den / d, targets, residual
WORDS_3D = 9  # persistent words per (member, obstacle, sample): alpha beta lx ly lz lca lsa lcb lsb


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=3)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--config", default="c5", choices=sorted(CONFIGS))
    ap.add_argument("--dtype", default="f64", choices=["f64", "f32"])
    ap.add_argument("--impl", default="b200", choices=["b200", "reference"])
    ap.add_argument("--groups", type=int, default=0)
    ap.add_argument("--layout", default=None, choices=["unit", "angle", "half"],
                    help="per-element state layout (unit: 11 words; angle: the reference's 9 words; half: 9 words, "
                         "angles as folded half-angle tangents)")
    ap.add_argument("--members", type=int, default=0, help="override the member count (testing)")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    a = ap.parse_args()
    if a.layout is None:  # the measured best for both storage types: half (the reference's 9 words)
        a.layout = "half"
    return a


def c4_problem():
    """C4 scene: 100 static spheres a = b = 0.4 (+5 cm) from default_rng(1),
    start (0,0,0) -> goal (12,0,0), v_max = a_max = 3, workspace box padded by 4, rho = 1."""
    from paper_2408_10731_b200 import scenarios, solver_priest
    from paper_2408_10731_b200.basis import AxisBoundary, build_basis, straight_line_coeffs

    basis = build_basis(0.0, 10.0, 100, 10)
    centers = scenarios.priest_c4_centers(100)
    specs = [scenarios.ObstacleSpec(0.4, 0.4, c, np.zeros(3)) for c in centers]
    obs = scenarios.tracks_on_grid(specs, basis.grid.timestamps)
    start, goal = np.zeros(3), np.array([12.0, 0.0, 0.0])
    pts = np.vstack([start, goal, centers])
    setup = solver_priest.ProjectionSetup(basis, tuple(AxisBoundary(p0=start[k], p1=goal[k]) for k in range(3)), obs,
                                          3.0, 3.0, pts.min(axis=0) - 4.0, pts.max(axis=0) + 4.0, 1.0)
    mean = straight_line_coeffs(basis, start, goal).ravel()
    dist = solver_priest.SamplingDistribution(mean, np.eye(mean.size) * 0.6**2)
    return setup, dist, solver_priest.BarnCost(start, goal)


def fp64_peak_tflops():
    import ctypes

    import torch

    from paper_2408_10731_b200 import _lib

    lib = _lib.load()
    scratch = torch.zeros(256, dtype=torch.float64, device="cuda")
    blocks = torch.cuda.get_device_properties(torch.cuda.current_device()).multi_processor_count * 8
    iters, best = 20000, 0.0
    for k in range(4):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        _lib.check(lib.tro_fp64_fma_probe(iters, blocks, scratch.data_ptr(), ctypes.c_void_p(_lib.stream_handle())),
                   "fp64 probe")
        b.record()
        torch.cuda.synchronize()
        if k:
            best = max(best, blocks * 256 * iters * 16 / (a.elapsed_time(b) / 1e3) / 1e12)
    return best


def run_c4(args):
    import torch
    import torch.distributed as tdist

    from paper_2408_10731_b200 import solver_priest as SP

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    if world > 1:
        tdist.init_process_group("nccl", device_id=torch.device("cuda", local))
    setup, dist, c1 = c4_problem()
    n_o, N, n_inner, desc = CONFIGS["c4"]
    params = SP.PriestParams(n_outer=C4_ROUNDS, n_batch=N, n_constraint_elite=C4_NCE, n_elite=C4_NEL,
                             n_inner=n_inner, seed=0)
    rng = np.random.default_rng(params.seed)
    z_host = np.stack([rng.standard_normal((N, dist.mu.size)) for _ in range(C4_ROUNDS)])  # the sampler's stream
    z_dev = torch.as_tensor(z_host, device="cuda")
    z_pin = torch.as_tensor(z_host).pin_memory()
    # one GPU: the single-device rounds; N GPUs: sample shards + one candidate all-gather per round
    opt = SP.priest_optimize if world == 1 else SP.priest_optimize_sharded

    def timed(fn):
        if world > 1:
            tdist.barrier()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        for _ in range(args.steps):
            out = fn()
        b.record()
        torch.cuda.synchronize()
        t = torch.tensor([a.elapsed_time(b) / 1e3 / args.steps], dtype=torch.float64, device="cuda")
        if world > 1:
            tdist.all_reduce(t, op=tdist.ReduceOp.MAX)
        return float(t.item()), out

    # one GPU: throughput mode: every round's draw factor (Cholesky) and standard normals
    # (Philox) are made on the device INSIDE the timed region; N GPUs: numpy-stream shards (parity mode)
    if world == 1:
        run_opt = lambda: SP.priest_optimize(setup, c1, dist, params, sampler="philox")  # noqa: E731
    else:
        run_opt = lambda: opt(setup, c1, dist, params, z_rounds=z_dev)  # noqa: E731
    for _ in range(args.warmup):
        run_opt()
    torch.cuda.synchronize()
    clocks = ClockSampler(local)
    clocks.start()
    step_s, res = timed(run_opt)
    clk = clocks.stop()
    # e2e: the public call with host inputs and host results (priest_optimize returns numpy mu, Sigma, best
    # sample, history); parity mode additionally uploads the reference sampler's normals from pinned memory
    e2e_s, res = timed(run_opt)
    parity_s, _ = timed(lambda: opt(setup, c1, dist, params, z_rounds=z_pin))
    # dominant kernel (projection) alone, CUDA events on its stream
    d = setup.device()
    d["L"].copy_(torch.as_tensor(SP._draw_factor(dist.sigma_mat)))
    d["mu"].copy_(torch.as_tensor(dist.mu))
    z_shard = z_dev[0][rank * (N // world):(rank + 1) * (N // world)].contiguous()
    SP._run_project(setup, z=z_shard, n_inner=n_inner)
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(3):
        SP._run_project(setup, z=z_shard, n_inner=n_inner)
    b.record()
    torch.cuda.synchronize()
    kern_s = a.elapsed_time(b) / 1e3 / 3
    n_loc = N // world
    flops = 32.0 * n_loc * n_o * 100 * n_inner  # 32 flop per sample-obstacle-timestep-inner-it
    peak = fp64_peak_tflops()
    value = N * n_inner * C4_ROUNDS / step_s
    line = {
        "metric": "sample-inner-iterations/sec (PRIEST projection, CEM rounds)",
        "value": value, "unit": "sample-inner-it/s", "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": step_s * 1e3, "ms_per_round": step_s * 1e3 / C4_ROUNDS, "higher_is_better": True,
        "scaling": "strong", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic (seeded C4 scene; throughput-mode Philox normals drawn on the device each round)",
        "config": {"workload": desc, "samples": N, "n_obs": n_o, "n_p": 100, "n_inner": n_inner,
                   "rounds": C4_ROUNDS, "constraint_elites": C4_NCE, "elites": C4_NEL, "l2": "on-chip (FP-bound)",
                   "parallelism": f"sample-shard x{world} (+ candidate all-gather / round)"},
        "roofline": {"bound": "fp64", "achieved": flops / kern_s / 1e12, "peak": peak, "unit": "TFLOP/s",
                     "frac": flops / kern_s / 1e12 / peak, "traffic": traffic_for("c4") if world == 1 else None,
                     "peak_source": "measured (tro_fp64_fma_probe, DFMA chains)",
                     "kernel": "tro_priest_project_f64 (priest_project_kernel<3>)",
                     "avg_launch_ms": kern_s * 1e3, "algorithmic_flops_per_launch": flops},
        "clocks": clk,
        "e2e": {"value": N * n_inner * C4_ROUNDS / e2e_s, "unit": "sample-inner-it/s",
                "h2d_bytes_per_step": int(8 * (33 * 33 + 33)),
                "d2h_bytes_per_step": int(8 * (33 * 33 + 33 + 3 * C4_ROUNDS + 2 * 33)),
                "api": "solver_priest.priest_optimize(..., sampler='philox')"},
        "parity_mode": {"value": N * n_inner * C4_ROUNDS / parity_s, "unit": "sample-inner-it/s",
                        "note": "numpy Generator normals (the reference's samples) uploaded from pinned host memory "
                                "every round, svd draw factor on the host",
                        "h2d_bytes_per_step": int(z_host.nbytes)},
        # per round: Cholesky, normals, projection, 2 x (order keys + rank select), aug cost, refit
        "gpu_launches": args.steps * C4_ROUNDS * (9 if world == 1 else 5),
        "result": {"best_aug_cost": res.history[-1]["best_aug_cost"], "best_residual": res.best.residual},
    }
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        v, info = cpu_reference_c4()
        line["cpu_baseline"] = {"value": v, "unit": "sample-inner-it/s", "cores": info["cores"], "kind": "port", "cpu_model": _cpu_model(),
                                "sample": info["sample"]}
    if rank == 0:
        print(json.dumps(line), flush=True)
    if world > 1:
        tdist.destroy_process_group()


def c3_problems(lo, hi):
    from paper_2408_10731_b200 import scenarios
    from paper_2408_10731_b200 import solver_multiagent as MA
    from paper_2408_10731_b200.basis import AxisBoundary, build_basis
    from paper_2408_10731_b200.geometry import EllipsoidShape

    b = build_basis(0.0, 10.0, 100, 10)
    probs = []
    for s in range(lo, hi):
        starts, goals = scenarios.square_antipodal(16, 8.0, 0.3, seed=s)
        bnds = [tuple(AxisBoundary(p0=float(starts[i, k]), p1=float(goals[i, k])) for k in range(3))
                for i in range(16)]
        probs.append(MA.MultiAgentProblem(basis=b, boundaries=bnds, agent_shape=EllipsoidShape(0.3, 0.45)))
    return probs


def b2_flops_per_member_iter(m=11, n_p=100, n_c=1, n_o=50):
    """Algorithmic fp64 flops of one batch_iteration of one member in the reference's formulation
    (Alg. 2 roofline): xi QP, heading contraction + QP, geometry, elements, F' contractions."""
    nv, nk = 4 * m, 4 * m + 12
    return (2 * nv * nk + 2 * m * n_p + 2 * m * (m + 2) + 2 * m * n_p * 10
            + B2_FLOPS_ELEM * n_c * n_o * n_p + 2 * m * n_p * 17)


def run_c2alt(args):
    import torch
    import torch.distributed as dist

    from paper_2408_10731_b200 import scenarios
    from paper_2408_10731_b200 import solver_batch as SB
    from paper_2408_10731_b200.distributed import shard_range, solve_batch_opt_sharded

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    if world > 1:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    n_o, total, n_iter, desc = CONFIGS["c2alt"]
    if args.members:
        total = args.members
    prob = scenarios.batch2d_problem(n_o=n_o, n_batch=total)
    params = SB.BatchParams(max_iter=n_iter)
    struct = SB._structure_for(prob)
    samples = SB._default_samples(prob, struct.m, None, None, 0)
    lo, hi = shard_range(total, rank, world)
    state0 = SB.init_state(prob, samples[lo:hi], params)
    lv = SB._levels(struct, 1.0, 1.0, params.rho_growth, params.rho_cap)
    eng = SB._Engine(struct, hi - lo, lv, params=params, max_hist=n_iter, member_offset=lo if world > 1 else None)
    gathered = torch.zeros((world, 4), dtype=torch.float64, device="cuda")
    stream = torch.cuda.current_stream()

    def iterations(n):
        if world == 1:
            eng.run(n)  # CUDA graphs of 25 launches; the last CTA applies the batch-global rule
            return
        for _ in range(n):  # batch-global rule across ranks: 32 B all-gather per iteration
            eng.iterate()
            dist.all_gather_into_tensor(gathered, eng.shard)
            eng.merge(gathered)

    def solve():
        eng.load(state0, 0)
        eng.prime(False)
        iterations(n_iter)
        eng.run_mode(3, eng.flags)

    for _ in range(args.warmup):
        solve()
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    clocks = ClockSampler(local)
    clocks.start()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record(stream)
    for _ in range(args.steps):
        solve()
    b.record(stream)
    torch.cuda.synchronize()
    clk = clocks.stop()
    t = torch.tensor([a.elapsed_time(b) / 1e3], dtype=torch.float64, device="cuda")
    if world > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    step_s = float(t.item()) / args.steps
    # the iterate kernel alone, CUDA events on its stream (single GPU: graph-replayed launches)
    eng.load(state0, 0)
    eng.prime(False)
    iterations(25)
    torch.cuda.synchronize()
    if world == 1:
        a.record(stream)
        eng.run(n_iter)
        b.record(stream)
        torch.cuda.synchronize()
        launch_s = a.elapsed_time(b) / 1e3 / n_iter
    else:
        a.record(stream)
        for _ in range(n_iter):
            eng.iterate()
        b.record(stream)
        torch.cuda.synchronize()
        launch_s = a.elapsed_time(b) / 1e3 / n_iter
    # e2e: the public API (samples from the host, ranked solutions back)
    api = (lambda: SB.solve_batch_opt(prob, params, samples=samples)) if world == 1 else \
        (lambda: solve_batch_opt_sharded(prob, params, samples=samples))
    api()
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    a.record(stream)
    for _ in range(args.steps):
        ranked = api()
    b.record(stream)
    torch.cuda.synchronize()
    te = torch.tensor([a.elapsed_time(b) / 1e3], dtype=torch.float64, device="cuda")
    if world > 1:
        dist.all_reduce(te, op=dist.ReduceOp.MAX)
    e2e_s = float(te.item()) / args.steps
    h2d = 8 * (hi - lo) * (4 * struct.m + struct.m + 100 + 4 * struct.m + struct.m) + 20
    d2h = 8 * (hi - lo) * (4 * struct.m + struct.m + 100 + 4 * struct.m + struct.m + 6) + 8 * 4 * n_iter + 20
    flops = b2_flops_per_member_iter(n_o=n_o) * (hi - lo)
    peak = fp64_peak_tflops()
    line = {
        "metric": "trajectory-iterations/sec (Alg. 2 batch x iterations)",
        "value": total * n_iter / step_s, "unit": "traj-it/s", "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": step_s * 1e3, "higher_is_better": True, "scaling": "strong",
        "vs_baseline": None, "dtype": "f64",
        "data": "synthetic (reference dynamic-flow generator, seed 0; default solve_batch_opt samples, seed 0)",
        "config": {"workload": desc, "members": total, "n_obs": n_o, "n_c": 1, "n_p": 100, "iterations": n_iter,
                   "parallelism": f"member-shard x{world} (+ 32 B all-gather / iteration)" if world > 1 else
                   "member-shard x1", "l2": "on-chip (latency-bound: state 1 MB, tracks 80 KB)"},
        "roofline": {"bound": "fp64", "achieved": flops / launch_s / 1e12, "peak": peak, "unit": "TFLOP/s",
                     "frac": flops / launch_s / 1e12 / peak, "traffic": traffic_for("c2alt") if world == 1 else None,
                     "peak_source": "measured (tro_fp64_fma_probe, DFMA chains)",
                     "kernel": "tro_b2_run mode 0 (b2_kernel<1, 0, circles>)", "avg_launch_ms": launch_s * 1e3,
                     "algorithmic_flops_per_launch": flops,
                     "note": "reference-formulation flops (bench.b2_flops_per_member_iter); the kernel is latency-"
                             "bound at 1024 members (7 per SM) and skips the closed forms of clamp-inactive circles"},
        "clocks": clk,
        "e2e": {"value": total * n_iter / e2e_s, "unit": "traj-it/s", "h2d_bytes_per_step": int(h2d),
                "d2h_bytes_per_step": int(d2h)},
        "gpu_launches": args.steps * (n_iter * (1 if world == 1 else 2) + 2),
        "result": {"best_index": ranked.best_index, "feasible": int(ranked.feasible.sum()),
                   "min_residual_max": float(ranked.residual_max.min()), "rho": ranked.state.rho},
    }
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        v, info = cpu_reference_c2alt()
        line["cpu_baseline"] = {"value": v, "unit": "traj-it/s", "cores": info["cores"], "kind": "port", "cpu_model": _cpu_model(),
                                "sample": info["sample"]}
    if rank == 0:
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()


def val_inputs(total: int):
    """C5 obstacles (raw shapes, no planning inflation) and member trajectories (straight-line coefficients)."""
    from paper_2408_10731_b200 import scenarios
    from paper_2408_10731_b200.basis import build_basis, line_basis_vectors

    basis = build_basis(0.0, 10.0, 100, 10)
    specs = scenarios.flow3d_obstacles(100)
    starts, goals = scenarios.flow3d_endpoints(range(total))
    u, v = line_basis_vectors(basis)
    xi = starts[:, :, None] * u[None, None, :] + (goals - starts)[:, :, None] * v[None, None, :]  # (B, 3, m)

    class Obs:
        def __init__(self, sp):
            self.a, self.b, self.center, self.velocity = sp.a, sp.b, list(sp.center), list(sp.velocity)

    class Scene:
        dim = 3
        obstacles = [Obs(sp) for sp in specs]

    return basis, Scene(), xi


def run_val(args):
    """N > 1: the trajectories shard into contiguous ranges, no collective on the data path."""
    import torch
    import torch.distributed as dist

    from paper_2408_10731_b200 import metrics as MT
    from paper_2408_10731_b200.distributed import shard_range

    world, rank, local = _dist_setup()
    n_o, total, _, desc = CONFIGS["val"]
    if args.members:
        total = args.members
    basis, sc, xi_all = val_inputs(total)
    lo, hi = shard_range(total, rank, world)
    xi = np.ascontiguousarray(xi_all[lo:hi])
    t = basis.grid.timestamps
    dev = torch.device("cuda")
    xi_dev = torch.as_tensor(xi, device=dev).contiguous()
    xi_pin = torch.as_tensor(xi).pin_memory()
    for _ in range(args.warmup):
        MT.validate_batch(sc, t, xi=xi_dev, basis=basis, return_device=True)
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    clocks = ClockSampler(local)
    clocks.start()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(args.steps):  # device-resident coefficients and results
        MT.validate_batch(sc, t, xi=xi_dev, basis=basis, return_device=True)
    b.record()
    torch.cuda.synchronize()
    clk = clocks.stop()
    step_s = _max_over_ranks(a.elapsed_time(b) / 1e3 / args.steps, world)
    for _ in range(args.warmup):  # the e2e path's own warm-up (pinned result buffer, copy stream)
        MT.validate_batch(sc, t, xi=xi_pin, basis=basis)
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    a.record()
    for _ in range(args.steps):
        r = MT.validate_batch(sc, t, xi=xi_pin, basis=basis)  # coefficients from pinned host memory, results back
    b.record()
    torch.cuda.synchronize()
    e2e_s = _max_over_ranks(a.elapsed_time(b) / 1e3 / args.steps, world)
    n_free = int(_sum_over_ranks(float(r["success"].sum()), world))
    flops = VAL_FLOPS_ELEM * total * n_o * 100
    peak = fp64_peak_tflops()
    line = {
        "metric": "trajectories validated/sec (raw-geometry metrics + collision check)", "value": total / step_s,
        "unit": "traj/s", "n_gpus": world, "steps": args.steps, "warmup": args.warmup, "ms_per_step": step_s * 1e3,
        "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic (C5 recipe obstacles, straight-line member trajectories)",
        "config": {"workload": desc, "members": total, "n_obs": n_o, "n_p": 100,
                   "parallelism": f"trajectory-shard x{world}"},
        "roofline": {"bound": "fp64", "achieved": flops / world / step_s / 1e12, "peak": peak, "unit": "TFLOP/s",
                     "frac": flops / world / step_s / 1e12 / peak,
                     "traffic": traffic_for("val") if world == 1 else None,
                     "peak_source": "measured (tro_fp64_fma_probe, DFMA chains)", "kernel": "tro_validate_f64",
                     "avg_launch_ms": step_s * 1e3, "algorithmic_flops_per_launch": flops,
                     "note": "per-step time includes validate_batch's host-side argument setup (cached constants)"},
        "clocks": clk,
        "e2e": {"value": total / e2e_s, "unit": "traj/s", "h2d_bytes_per_step": int(xi_all.nbytes),
                "d2h_bytes_per_step": int(total * 5 * 8)},
        "gpu_launches": args.steps,
        "result": {"collision_free": n_free},
    }
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        v, info = cpu_reference_val()
        line["cpu_baseline"] = {"value": v, "unit": "traj/s", "cores": 1, "kind": "port", "cpu_model": _cpu_model(), "sample": info}
    if rank == 0:
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()


def cpu_reference_val(n_s=64):
    """The oracle port of bench.metrics on a bounded sample of the validation workload (1 core)."""
    from oracle import metrics as OMT

    basis, sc, xi = val_inputs(n_s)
    t = basis.grid.timestamps
    c = np.array([o.center for o in sc.obstacles])
    v = np.array([o.velocity for o in sc.obstacles])
    aa = np.array([o.a for o in sc.obstacles])
    bb = np.array([o.b for o in sc.obstacles])
    t0 = time.perf_counter()
    for k in range(n_s):
        OMT.metrics(basis.P @ xi[k].T, basis.Pddot @ xi[k].T, t, c, v, aa, bb, 3)
    wall = time.perf_counter() - t0
    return n_s / wall, f"{n_s} trajectories x 100 obstacles, oracle port of bench.metrics (1 core)"


def _dist_setup():
    """(world, rank, local) with the NCCL process group initialised for N > 1 (one process per GPU)."""
    import torch
    import torch.distributed as dist

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    if world > 1:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    return world, rank, local


def _max_over_ranks(x: float, world: int) -> float:
    import torch
    import torch.distributed as dist

    if world == 1:
        return x
    t = torch.tensor([x], dtype=torch.float64, device="cuda")
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def _sum_over_ranks(x: float, world: int) -> float:
    import torch
    import torch.distributed as dist

    if world == 1:
        return x
    t = torch.tensor([x], dtype=torch.float64, device="cuda")
    dist.all_reduce(t, op=dist.ReduceOp.SUM)
    return float(t.item())


def mpc_inputs(total: int):
    """The C2 obstacle field as a bench Scenario (3-D, a 0.4 / b 0.3, seeded recipe) + C2 member endpoints."""
    from paper_2408_10731_b200 import scenarios
    from paper_2408_10731_b200.bench import scenarios as SC

    specs = scenarios.flow3d_obstacles(CONFIGS["mpc"][0])
    starts, goals = scenarios.flow3d_endpoints(range(total))
    sc = SC.Scenario(kind="dynamic-flow", dim=3, horizon=SC.Horizon(t0=0.0, tf=10.0, n_p=100),
                     robot=SC.RobotSpec(shape=[0.0, 0.0], v_max=3.0, a_max=3.0),
                     obstacles=[SC.ScenarioObstacle(a=o.a, b=o.b, center=[float(x) for x in o.center],
                                                    velocity=[float(x) for x in o.velocity]) for o in specs],
                     boundary=SC.Boundary(start=[0.0, 0.0, 0.0], goal=[12.0, 0.0, 0.0]), seed=0)
    return sc, starts, goals


def run_mpc(args):
    """One step = one receding-horizon episode of the whole fleet (30 control steps of 40 warm AM iterations
    + predict / validate / advance per control step), device-resident between control steps.  N > 1: the
    robots shard into contiguous ranges (no collective on the data path: robots are independent)."""
    import torch
    import torch.distributed as dist

    from paper_2408_10731_b200.distributed import shard_range
    from paper_2408_10731_b200.mpc import MpcFleet

    world, rank, local = _dist_setup()
    n_o, total, budget, desc = CONFIGS["mpc"]
    if args.members:
        total = args.members
    sc, starts_all, goals_all = mpc_inputs(total)
    lo, hi = shard_range(total, rank, world)
    starts, goals = starts_all[lo:hi], goals_all[lo:hi]
    fleet = MpcFleet(sc, starts, goals, step_budget=budget, layout=args.layout)
    for _ in range(args.warmup):
        fleet.run(MPC_STEPS, early_exit=False)
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    clocks = ClockSampler(local)
    clocks.start()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    solve_ms = []
    a.record()
    for _ in range(args.steps):
        fr = fleet.run(MPC_STEPS, early_exit=False)
        solve_ms.append(float(fr.step_ms.sum()))
    b.record()
    torch.cuda.synchronize()
    clk = clocks.stop()
    step_s = _max_over_ranks(a.elapsed_time(b) / 1e3 / args.steps, world)
    # robots that collided or reached the goal are frozen (no further solves): count the control steps solved
    robot_steps = int(_sum_over_ranks(float(sum(fr.steps_of(i) for i in range(hi - lo))), world))
    # e2e: the public API from host arrays: fleet construction (uploads) + episode + results to the host
    if world > 1:
        dist.barrier()
    t0 = time.perf_counter()
    for _ in range(args.steps):
        fr_e = MpcFleet(sc, starts, goals, step_budget=budget, layout=args.layout).run(MPC_STEPS, early_exit=False)
    e2e_s = _max_over_ranks((time.perf_counter() - t0) / args.steps, world)
    flags = [int((fr.flags == k).sum()) for k in (0, 1, 2)]
    flags = [int(_sum_over_ranks(float(f), world)) for f in flags]
    # roofline of the dominant kernel (the fused AM iteration): algorithmic bytes per launch / per-iteration time
    it_ms = _max_over_ranks(statistics.mean(solve_ms) / MPC_STEPS / budget, world)
    bytes_launch = 2 * WORDS_3D * n_o * 100 * 8 * robot_steps / MPC_STEPS / world  # mean active robots per launch
    peak, peak_src = measured_peaks()
    line = {
        "metric": "robot control steps/sec (receding horizon, 40 warm AM its per step)",
        "value": robot_steps / step_s, "unit": "robot-steps/s", "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": step_s * 1e3, "higher_is_better": True, "scaling": "strong",
        "vs_baseline": None, "dtype": "f64", "data": "synthetic (C2 recipe obstacle field and endpoints)",
        "config": {"workload": desc, "robots": total, "n_obs": n_o, "n_p": 100, "control_steps": MPC_STEPS,
                   "step_budget": budget, "layout": args.layout, "parallelism": f"robot-shard x{world}",
                   "l2": "per-element state 368 MB > L2"},
        "control_step_ms": step_s * 1e3 / MPC_STEPS,
        "paper_budget_ms": 40.0,
        "roofline": {"bound": "hbm", "achieved": bytes_launch / (it_ms * 1e-3) / 1e9, "peak": peak, "unit": "GB/s",
                     "frac": bytes_launch / (it_ms * 1e-3) / 1e9 / peak,
                     "traffic": traffic_for("mpc") if world == 1 else None, "peak_source": peak_src,
                     "kernel": "alg1 fused AM iteration (incl. the per-step prime)",
                     "avg_launch_ms": it_ms, "algorithmic_bytes_per_launch": bytes_launch},
        "clocks": clk,
        "e2e": {"value": robot_steps / e2e_s, "unit": "robot-steps/s",
                "h2d_bytes_per_step": int(starts_all.nbytes + goals_all.nbytes),
                "d2h_bytes_per_step": int(fr_e.trace.nbytes + fr_e.metrics.nbytes + fr_e.residual.nbytes
                                          + fr_e.flags.nbytes + fr_e.n_trace.nbytes)},
        "gpu_launches": args.steps * (2 + MPC_STEPS * (4 + budget)),
        "result": {"still_driving": flags[0], "collided": flags[1], "reached": flags[2],
                   "robot_steps_solved": robot_steps, "robot_steps_offered": total * MPC_STEPS},
    }
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        v, info = cpu_reference_mpc()
        line["cpu_baseline"] = {"value": v, "unit": "robot-steps/s", "cores": 1, "kind": "port", "cpu_model": _cpu_model(),
                                "sample": info}
    if rank == 0:
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()


def cpu_reference_mpc(robots=2, steps=3):
    """The oracle port of receding_horizon_run (bit-exact with the reference) on a bounded sample."""
    from oracle import mpc as OM
    from paper_2408_10731_b200.basis import build_basis
    from paper_2408_10731_b200.bench.scenarios import obstacle_arrays

    sc, starts, goals = mpc_inputs(robots)
    b = build_basis(0.0, 10.0, 100, 10)
    c, v, aa, bb = obstacle_arrays(sc)
    t0 = time.perf_counter()
    OM.run(b.P, b.Pdot, b.Pddot, b.grid.timestamps, c, v, aa, bb, starts, goals, step_budget=CONFIGS["mpc"][2],
           n_steps=steps)
    wall = time.perf_counter() - t0
    return robots * steps / wall, f"{robots} robots x {steps} control steps x 40 AM its (oracle port, 1 core)"


def cpu_reference_c2alt(n_iter=3):
    """Oracle port of solve_batch_opt (bit-exact with the reference) on the full batch, all BLAS threads:
    the reference is numpy-vectorised over the batch (solver_batch.py:352-363)."""
    from oracle import batch2d as OB
    from paper_2408_10731_b200 import scenarios
    from paper_2408_10731_b200 import solver_batch as SB

    n_o, total, _, _ = CONFIGS["c2alt"]
    prob = scenarios.batch2d_problem(n_o=n_o, n_batch=total)
    b = prob.basis
    st = OB.make_structure(b.P, b.Pdot, b.Pddot, np.stack([bc.values() for bc in prob.boundary]), prob.psi_boundary,
                           prob.desired, np.stack([o.centers for o in prob.obstacles]),
                           [o.shape.a for o in prob.obstacles], [o.shape.b for o in prob.obstacles], (0.0,), 3.0, 3.0)
    samples = SB._default_samples(prob, b.n_var, None, None, 0)
    OB.solve(st, samples[:8], 1, max_iter=1)
    t0 = time.perf_counter()
    OB.solve(st, samples, 1, max_iter=n_iter)
    wall = time.perf_counter() - t0
    cores = os.cpu_count() or 1
    return total * n_iter / wall, {"cores": cores, "sample": f"{total} members x {n_iter} iterations (init + "
                                                             f"ranking included), oracle port, numpy/BLAS "
                                                             f"threads, wall {wall:.1f}s"}


def run_c3(args):
    import torch
    import torch.distributed as dist

    from paper_2408_10731_b200 import solver_multiagent as MA
    from paper_2408_10731_b200.distributed import gather_summaries, shard_range, shard_summary

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    if world > 1:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    n_a, total, n_iter, desc = CONFIGS["c3"]
    if args.members:
        total = args.members
    lo, hi = shard_range(total, rank, world)
    probs = c3_problems(lo, hi)
    params = MA.JointParams(max_iter=n_iter, rho_final=1e3, tol_norm=0.0)
    struct = MA._Structure(probs[0], params)
    b_eq = np.stack([MA._b_eq(p) for p in probs])
    eng = MA.MaEngine(struct, b_eq, None, params)
    stream = torch.cuda.current_stream()

    def solve():
        eng.reset()
        eng.init()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        eng.run(n_iter, use_graph=True, check_every=0)
        e1.record(stream)
        return e0, e1

    for _ in range(args.warmup):
        solve()
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    clocks = ClockSampler(local)
    clocks.start()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    runs = []
    a.record(stream)
    for _ in range(args.steps):
        runs.append(solve())
        if world > 1:
            gather_summaries(shard_summary(eng.res_max, eng.res_norm, eng.res_norm <= 0.01, lo))
    b.record(stream)
    torch.cuda.synchronize()
    clk = clocks.stop()
    t = torch.tensor([a.elapsed_time(b) / 1e3], dtype=torch.float64, device="cuda")
    if world > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    elapsed = float(t.item())
    launch_s = statistics.mean(x.elapsed_time(y) for x, y in runs) / 1e3 / n_iter
    n_pairs = struct.n_pairs
    # W = 4 persistent words per pair-sample (lambda x/y/z and d) -> 768 KB per problem-iteration;
    # this kernel keeps 3 (d is folded into the agent sums), so it moves 3/4 of the algorithmic bytes
    alg_bytes = 2 * 4 * n_pairs * 100 * 8 * (hi - lo)
    moved_bytes = 2 * 3 * n_pairs * 100 * 8 * (hi - lo)
    peak, peak_src = measured_peaks()
    # e2e: boundary values from pinned host memory each step, xi / residuals back
    bv_pin = torch.as_tensor(b_eq).pin_memory()
    xi_pin = torch.empty(eng.xi.shape, dtype=torch.float64).pin_memory()
    r_pin = torch.empty((2, eng.B), dtype=torch.float64).pin_memory()
    a.record(stream)
    for _ in range(args.steps):
        eng.b_eq.copy_(bv_pin, non_blocking=True)
        solve()
        xi_pin.copy_(eng.xi, non_blocking=True)
        r_pin[0].copy_(eng.res_norm, non_blocking=True)
        r_pin[1].copy_(eng.res_max, non_blocking=True)
    b.record(stream)
    torch.cuda.synchronize()
    te = torch.tensor([a.elapsed_time(b) / 1e3], dtype=torch.float64, device="cuda")
    if world > 1:
        dist.all_reduce(te, op=dist.ReduceOp.MAX)
    line = {
        "metric": "problem-iterations/sec (joint 16-agent problems x iterations)",
        "value": total * n_iter * args.steps / elapsed, "unit": "problem-it/s",
        "agent_traj_it_per_s": 16 * total * n_iter * args.steps / elapsed,
        "n_gpus": world, "steps": args.steps, "warmup": args.warmup, "ms_per_step": elapsed / args.steps * 1e3,
        "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic (square-antipodal rosters, seeds 0..4095)",
        "config": {"workload": desc, "problems": total, "agents": 16, "pairs": n_pairs, "n_p": 100,
                   "iterations": n_iter, "parallelism": f"problem-shard x{world}", "l2": "state >> L2"},
        "roofline": {"bound": "hbm", "achieved": alg_bytes / launch_s / 1e9, "peak": peak, "unit": "GB/s",
                     "frac": alg_bytes / launch_s / 1e9 / peak, "traffic": traffic_for("c3") if world == 1 else None,
                     "peak_source": peak_src,
                     "kernel": "tro_ma_run modes 3 + 4 (ma_qp_kernel<11>: DMMA QP; ma_kernel<11, 4>: element pass), per iteration", "avg_launch_ms": launch_s * 1e3,
                     "algorithmic_bytes_per_launch": alg_bytes, "state_bytes_moved_per_launch": moved_bytes,
                     "hbm_frac_of_moved_bytes": moved_bytes / launch_s / 1e9 / peak,
                     "note": "algorithmic = SURVEY 8(d) W = 4 words per pair-sample (lambda x/y/z, d); the kernel "
                             "moves 3 (d only feeds the next RHS and is folded into the agent sums)"},
        "clocks": clk,
        "e2e": {"value": total * n_iter * args.steps / float(te.item()), "unit": "problem-it/s",
                "h2d_bytes_per_step": int(b_eq.nbytes), "d2h_bytes_per_step": int(xi_pin.numel() * 8 + r_pin.numel() * 8)},
        "gpu_launches": args.steps * (n_iter * (2 if eng.split_qp else 1) + 1),
    }
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        v, info = cpu_reference_c3()
        line["cpu_baseline"] = {"value": v, "unit": "problem-it/s", "cores": info["cores"], "kind": "port", "cpu_model": _cpu_model(),
                                "sample": info["sample"]}
    if rank == 0:
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()


def _oracle_ma_solve(args):
    os.environ["OPENBLAS_NUM_THREADS"] = "1"
    seed, n_iter = args
    from oracle import multiagent as OM
    from paper_2408_10731_b200 import solver_multiagent as MA

    prob = c3_problems(seed, seed + 1)[0]
    b = prob.basis
    st = OM.make_structure(b.P, b.Pdot, b.Pddot, 16, 0.3, 0.45, rho_final=1e3)
    t0 = time.perf_counter()
    OM.solve(st, OM.Problem(b_eq=MA._b_eq(prob), statics=np.zeros((0, 3))), b.P, max_iter=n_iter, tol_norm=0.0)
    return time.perf_counter() - t0


def cpu_reference_c3(procs=None, n_iter=200):
    """Oracle port of solve_joint (bit-exact with the reference), one problem per core."""
    import multiprocessing as mp

    procs = procs or os.cpu_count() or 1
    ctx = mp.get_context("spawn")
    with ctx.Pool(procs) as pool:
        pool.map(_oracle_ma_solve, [(0, 1)] * procs)
        t0 = time.perf_counter()
        pool.map(_oracle_ma_solve, [(s, n_iter) for s in range(procs)], chunksize=1)
        wall = time.perf_counter() - t0
    return procs * n_iter / wall, {"cores": procs, "sample": f"{procs} C3 problems x {n_iter} iterations, "
                                                             f"oracle port (1 BLAS thread), wall {wall:.1f}s"}


def _oracle_project_chunk(args):
    os.environ["OPENBLAS_NUM_THREADS"] = "1"
    lo, hi, n_inner = args
    from oracle import priest as OP

    setup, dist, _ = c4_problem_host()
    rng = np.random.default_rng(0)
    z = rng.standard_normal((16384, dist[0].size))[lo:hi]
    samples = dist[0] + z @ OP.draw_transform(dist[0], dist[1]).T
    t0 = time.perf_counter()
    OP.project(setup, samples, n_inner)
    return time.perf_counter() - t0


def c4_problem_host():
    """The C4 scene as oracle arrays (no GPU needed)."""
    from oracle import priest as OP
    from paper_2408_10731_b200 import scenarios
    from paper_2408_10731_b200.basis import build_basis, straight_line_coeffs

    basis = build_basis(0.0, 10.0, 100, 10)
    centers = scenarios.priest_c4_centers(100)
    tracks = np.repeat(centers[:, None, :], 100, axis=1)
    start, goal = np.zeros(3), np.array([12.0, 0.0, 0.0])
    pts = np.vstack([start, goal, centers])
    bvals = np.zeros((3, 6))
    bvals[:, 0], bvals[:, 3] = start, goal
    st = OP.make_setup(basis.P, basis.Pdot, basis.Pddot, bvals, tracks, np.full(100, 0.45), np.full(100, 0.45), 3.0,
                       3.0, pts.min(axis=0) - 4.0, pts.max(axis=0) + 4.0, 1.0)
    mean = straight_line_coeffs(basis, start, goal).ravel()
    return st, (mean, np.eye(mean.size) * 0.36), None


def cpu_reference_c4(procs=None, per_proc=8, n_inner=30):
    """Reference CPU projection (oracle port of solver_priest.project, bit-exact with the reference
    on the golden rounds) on a bounded sample: per_proc samples per core, all cores."""
    import multiprocessing as mp

    procs = procs or os.cpu_count() or 1
    ctx = mp.get_context("spawn")
    tasks = [(k * per_proc, (k + 1) * per_proc, n_inner) for k in range(procs)]
    with ctx.Pool(procs) as pool:
        pool.map(_oracle_project_chunk, [(0, 1, 1)] * procs)
        t0 = time.perf_counter()
        pool.map(_oracle_project_chunk, tasks, chunksize=1)
        wall = time.perf_counter() - t0
    n = procs * per_proc
    return n * n_inner / wall, {"cores": procs, "sample": f"{n} C4 samples x {n_inner} inner its (one round's "
                                                          f"projection slice), oracle port, wall {wall:.1f}s"}


def _alg1_loop_max() -> int:
    from paper_2408_10731_b200 import _alg1

    return _alg1.LOOP_MAX_MEMBERS


def traffic_for(cfg: str):
    """dram__bytes_read + dram__bytes_write of one launch of the config's dominant kernel, from the committed
    ncu capture (profiles/ncu_traffic_r1.json, tools/ncu_traffic.sh); None when absent."""
    path = os.path.join(ROOT, "profiles", "ncu_traffic_r1.json")
    if not os.path.exists(path):
        return None
    with open(path) as fh:
        d = json.load(fh)
    return d.get(cfg, {}).get("dram_bytes_per_launch")


def _cpu_model() -> str:
    """The host CPU the baseline ran on (BASELINE.md §3 asks for it), from /proc/cpuinfo."""
    try:
        with open("/proc/cpuinfo") as fh:
            for line in fh:
                if line.startswith("model name"):
                    return line.split(":", 1)[1].strip()
    except OSError:
        pass
    import platform

    return platform.processor() or "unknown"


def measured_peaks():
    path = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(path):
        with open(path) as fh:
            d = json.load(fh)
        return float(d["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs)"
    return 6650.0, "fallback (B200_PROFILING.md 6.65 TB/s)"


# ---------------------------------------------------------------- clocks sampling
class ClockSampler:
    """SM clocks and throttle reasons sampled DURING the timed region: NVML polled every 5 ms from a
    thread (short regions still get samples); nvidia-smi -lms 200 when NVML is unavailable."""

    FIELDS = ("clocks.sm,clocks.max.sm,clocks_event_reasons.active,clocks_event_reasons.hw_slowdown,"
              "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
              "clocks_event_reasons.sw_power_cap")
    NAMES = ("hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap")

    def __init__(self, index: int):
        self.index = index
        self.rows = []
        self.proc = None
        self.nvml = None
        self._stop = threading.Event()

    def start(self):
        try:
            import pynvml

            pynvml.nvmlInit()
            vis = os.environ.get("CUDA_VISIBLE_DEVICES")
            idx = int(vis.split(",")[self.index]) if vis and vis.split(",")[0].isdigit() else self.index
            h = pynvml.nvmlDeviceGetHandleByIndex(idx)
            self.nvml = (pynvml, h)
            self.max_mhz = pynvml.nvmlDeviceGetMaxClockInfo(h, pynvml.NVML_CLOCK_SM)
            masks = (pynvml.nvmlClocksEventReasonHwSlowdown, pynvml.nvmlClocksEventReasonHwThermalSlowdown,
                     pynvml.nvmlClocksEventReasonSwThermalSlowdown, pynvml.nvmlClocksEventReasonSwPowerCap)

            def poll():
                while not self._stop.is_set():
                    sm = pynvml.nvmlDeviceGetClockInfo(h, pynvml.NVML_CLOCK_SM)
                    r = pynvml.nvmlDeviceGetCurrentClocksEventReasons(h)
                    self.rows.append((sm, tuple(bool(r & mk) for mk in masks)))
                    time.sleep(0.005)

            self.thread = threading.Thread(target=poll, daemon=True)
            self.thread.start()
            return
        except Exception:  # noqa: BLE001 - fall back to nvidia-smi
            self.nvml = None
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.FIELDS}", "--format=csv,noheader,nounits",
                 "-lms", "200"], stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.thread = threading.Thread(target=self._read, daemon=True)
            self.thread.start()
        except OSError:
            self.proc = None

    def _read(self):
        for line in self.proc.stdout:
            parts = [p.strip() for p in line.split(",")]
            if len(parts) >= 7:
                self.rows.append(parts)

    def stop(self):
        if self.nvml is not None:
            self._stop.set()
            self.thread.join(timeout=1)
            sm = [float(r[0]) for r in self.rows]
            reasons = sorted({self.NAMES[k] for r in self.rows for k in range(4) if r[1][k]})
            return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": float(self.max_mhz),
                    "reasons": reasons, "samples": len(self.rows), "source": "nvml 5 ms"}
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except subprocess.TimeoutExpired:
            self.proc.kill()
        sm = [float(r[0]) for r in self.rows if r[0].replace(".", "").isdigit()]
        mx = [float(r[1]) for r in self.rows if r[1].replace(".", "").isdigit()]
        reasons = sorted({self.NAMES[k] for r in self.rows for k in range(4)
                          if "Active" in r[3 + k] and r[3 + k] != "Not Active"})
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": reasons, "samples": len(self.rows), "source": "nvidia-smi 200 ms"}


# ---------------------------------------------------------------- CPU reference arm (oracle port)
def _oracle_member_solve(args):
    os.environ["OPENBLAS_NUM_THREADS"] = "1"
    n_o, member, n_iter = args
    from oracle import alg1 as O
    from paper_2408_10731_b200 import scenarios
    from paper_2408_10731_b200.basis import build_basis

    bs = build_basis(0.0, 10.0, 100, 10)
    batch = scenarios.flow3d_batch(n_o, [member], basis=bs) if n_o != 10 else None
    if batch is None:
        prob = scenarios.c1_problem()
        tracks = np.stack([o.centers for o in prob.obstacles])
        bvals = np.stack([bc.values() for bc in prob.boundary])[None]
        desired = prob.desired[None]
        a = np.array([o.shape.a for o in prob.obstacles])
        b = np.array([o.shape.b for o in prob.obstacles])
    else:
        tracks = np.stack([o.centers for o in batch.obstacles])
        bvals = batch.bvals
        s = np.linspace(0, 1, 100)
        desired = bvals[:, :, 0][:, None, :] + s[None, :, None] * (bvals[:, :, 3] - bvals[:, :, 0])[:, None, :]
        a = np.array([o.shape.a for o in batch.obstacles])
        b = np.array([o.shape.b for o in batch.obstacles])
    prob = O.Problem(P=bs.P, Pd=bs.Pdot, Pdd=bs.Pddot, bvals=bvals, desired=desired, tracks=tracks, a=a, b=b)
    t0 = time.perf_counter()
    O.solve(prob, O.Params(max_iter=n_iter, tol=0.0))
    return time.perf_counter() - t0


def cpu_reference(cfg_name: str, members: int, procs: int | None = None):
    """Reference CPU path: the oracle port of solver_single (bit-exact with the reference on C1),
    one member per task, 1 BLAS thread per process, all host cores.  Returns (traj-it/s, info)."""
    import multiprocessing as mp

    n_o, _, n_iter, _ = CONFIGS[cfg_name]
    procs = procs or os.cpu_count() or 1
    ctx = mp.get_context("spawn")
    os.environ["OPENBLAS_NUM_THREADS"] = "1"
    tasks = [(n_o, i, n_iter) for i in range(members)]
    with ctx.Pool(procs) as pool:
        pool.map(_oracle_member_solve, [(n_o, 0, 2)] * procs)  # import warm-up
        t0 = time.perf_counter()
        pool.map(_oracle_member_solve, tasks, chunksize=1)
        wall = time.perf_counter() - t0
    return members * n_iter / wall, {"cores": procs, "wall_s": wall, "members": members, "iterations": n_iter}


# ---------------------------------------------------------------- GPU arm
def run_b200(args):
    import torch
    import torch.distributed as dist

    from paper_2408_10731_b200 import scenarios
    from paper_2408_10731_b200.basis import build_basis
    from paper_2408_10731_b200.distributed import gather_summaries, shard_range, shard_summary
    from paper_2408_10731_b200.solver_single import SingleBatch, SingleParams, make_batch_engine

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    if world > 1:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    n_o, members_total, n_iter, desc = CONFIGS[args.config]
    if args.members:
        members_total = args.members
    lo, hi = shard_range(members_total, rank, world)
    B = hi - lo
    dtype = torch.float64 if args.dtype == "f64" else torch.float32
    s_bytes = 8 if args.dtype == "f64" else 4

    basis = build_basis(0.0, 10.0, 100, 10)
    if args.config == "c1":
        batch = SingleBatch.from_problems([scenarios.c1_problem()])
    else:
        batch = scenarios.flow3d_batch(n_o, range(lo, hi), basis=basis)
    params = SingleParams(max_iter=n_iter, tol=0.0)
    eng = make_batch_engine(batch, params, dtype=dtype, groups=args.groups, layout=args.layout)
    stream = torch.cuda.current_stream()

    def solve_device():
        eng.cold_init()  # complete cold start on the device: rho, rho_o, level, iteration, schedule reset
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        eng.run(n_iter, use_graph=True)
        e1.record(stream)
        return e0, e1

    def summary():
        # per-shard end-of-solve summary (best member, converged count): the only collective
        return shard_summary(eng.res_max, eng.res_norm, eng.res_max <= 1e-3, lo)

    for _ in range(args.warmup):
        solve_device()
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    clocks = ClockSampler(local)
    clocks.start()
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    start = torch.cuda.Event(enable_timing=True)
    stop = torch.cuda.Event(enable_timing=True)
    iter_ms = []
    start.record(stream)
    for _ in range(args.steps):
        e0, e1 = solve_device()
        if world > 1:
            gather_summaries(summary())
        iter_ms.append((e0, e1))
    stop.record(stream)
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    clk = clocks.stop()
    elapsed = start.elapsed_time(stop) / 1e3
    run_ms = [a.elapsed_time(b) for a, b in iter_ms]
    t = torch.tensor([elapsed], dtype=torch.float64, device="cuda")
    if world > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    elapsed = float(t.item())
    value = members_total * n_iter * args.steps / elapsed

    # roofline of the dominant kernel (tro_alg1_iterate): ALGORITHMIC bytes per launch (the reference's
    # 9 persistent words per element) / avg launch time -- independent of the layout
    alg_bytes = 2 * WORDS_3D * n_o * 100 * s_bytes * B
    moved_bytes = 2 * eng.W * n_o * 100 * s_bytes * B
    avg_launch_s = statistics.mean(run_ms) / 1e3 / n_iter
    peak, peak_src = measured_peaks()
    achieved = alg_bytes / avg_launch_s / 1e9
    traffic = None
    # DRAM bytes per launch from the committed ncu --set full capture of the same kernel
    # (same layout / dtype), scaled from per-element bytes to this launch's element count
    tpath = os.path.join(ROOT, "profiles", f"ncu_alg1_{args.layout}_{args.dtype}.json")
    if os.path.exists(tpath):
        with open(tpath) as fh:
            prof = json.load(fh)
        traffic = prof.get("dram_bytes_per_element_launch", 0) * B * n_o * 100 or None

    # the last timed solve must be a cold solve: its first members equal a fresh engine's solve bitwise
    # (members are independent and run whole on one CTA; the fresh engine has no tail split)
    n_chk = min(B, 512)
    xi_last = eng.xi[:n_chk].clone()
    res_last = eng.res_max[:n_chk].clone()
    chk_batch = (SingleBatch.from_problems([scenarios.c1_problem()]) if args.config == "c1"
                 else scenarios.flow3d_batch(n_o, range(lo, lo + n_chk), basis=basis))
    chk = make_batch_engine(chk_batch, params, dtype=dtype, groups=args.groups, layout=args.layout,
                            tail_split=False)
    chk.cold_init()
    chk.run(n_iter, use_graph=True)
    fresh_equal = bool(torch.equal(chk.xi, xi_last) and torch.equal(chk.res_max, res_last))
    del chk
    torch.cuda.empty_cache()
    if not fresh_equal:
        raise SystemExit("bench: the last timed solve differs from a fresh-engine solve (stale state)")

    # e2e through the public API (solve_single_batch) with host numpy in and out: each step uploads the
    # members' boundary values, computes the linear terms on the device, cold-starts, runs the AM loop and
    # copies every per-member result back (xi, residuals, rho_o, flags, counters) in one D2H copy
    e2e = None
    if not args.no_e2e:
        from paper_2408_10731_b200.solver_single import solve_single_batch

        host_batch = SingleBatch(batch.basis, np.ascontiguousarray(batch.bvals), list(batch.obstacles),
                                 batch.desired, batch.w_smooth, batch.w_track)
        res = solve_single_batch(host_batch, params, engine=eng, use_graph=True).numpy()  # warm (graph built)
        h2d = host_batch.bvals.nbytes
        d2h = B * (eng.xi[0].numel() + 6) * 8
        torch.cuda.synchronize()
        if world > 1:
            dist.barrier()
        a = torch.cuda.Event(enable_timing=True)
        b = torch.cuda.Event(enable_timing=True)
        w0 = time.perf_counter()
        a.record(stream)
        for _ in range(args.steps):
            res = solve_single_batch(host_batch, params, engine=eng, use_graph=True).numpy()
        b.record(stream)
        torch.cuda.synchronize()
        wall_e2e = time.perf_counter() - w0
        te = torch.tensor([a.elapsed_time(b) / 1e3], dtype=torch.float64, device="cuda")
        if world > 1:
            dist.all_reduce(te, op=dist.ReduceOp.MAX)
        if not np.array_equal(res.xi[:n_chk], xi_last.cpu().numpy()):
            raise SystemExit("bench: the public-API solve differs from the device-timed solve")
        e2e = {"value": members_total * n_iter * args.steps / float(te.item()), "unit": "traj-it/s",
               "h2d_bytes_per_step": int(h2d), "d2h_bytes_per_step": int(d2h),
               "api": "solver_single.solve_single_batch(SingleBatch numpy in, engine=cached).numpy()",
               "wall_s": wall_e2e}
        if args.config == "c1" and world == 1:
            # C1 is the reference's single-problem case: the call a user makes is solve_single (numpy in,
            # SingleSolution out: trajectory, histories, state), timed on the stream around the call
            from paper_2408_10731_b200 import scenarios as _sc
            from paper_2408_10731_b200 import solver_single as _ss

            prob = _sc.c1_problem()
            prm = _ss.SingleParams(max_iter=n_iter, tol=0.0)
            _ss.solve_single(prob, prm)
            torch.cuda.synchronize()
            a.record(stream)
            for _ in range(args.steps):
                sol = _ss.solve_single(prob, prm)
            b.record(stream)
            torch.cuda.synchronize()
            e2e = {"value": n_iter * args.steps / (a.elapsed_time(b) / 1e3), "unit": "traj-it/s",
                   "h2d_bytes_per_step": int(h2d), "d2h_bytes_per_step": int(sol.state.xi.nbytes + 8 * 3 * n_iter),
                   "api": "solver_single.solve_single"}

    line = {
        "metric": "trajectory-iterations/sec (batch x AM iters)",
        "value": value,
        "unit": "traj-it/s",
        "n_gpus": world,
        "steps": args.steps,
        "warmup": args.warmup,
        "ms_per_step": elapsed / args.steps * 1e3,
        "higher_is_better": True,
        "scaling": "strong",
        "vs_baseline": None,
        "dtype": args.dtype,
        "data": "synthetic (seeded scenario recipe, SURVEY.md §8(d))",
        "config": {"workload": desc, "members": members_total, "n_obs": n_o, "n_p": 100, "am_iters": n_iter,
                   "state_dtype": args.dtype, "state_layout": args.layout, "qp_step": "f64",
                   "parallelism": f"member-shard x{world}",
                   "l2": "state >> L2 (no flush needed)" if alg_bytes > 126e6 else "state fits L2"},
        "roofline": {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s", "frac": achieved / peak,
                     "traffic": traffic, "peak_source": peak_src,
                     "algorithmic_bytes_per_launch": alg_bytes, "avg_launch_ms": avg_launch_s * 1e3,
                     "layout": args.layout, "state_bytes_moved_per_launch": moved_bytes,
                     "hbm_frac_of_moved_bytes": moved_bytes / avg_launch_s / 1e9 / peak,
                     "kernel": "tro_alg1_iterate (alg1_tma_kernel<3,T,LAY,100,G,MINB,2>: persistent, warp-"
                               "specialised producer / scalar / consumer warps)"},
        "clocks": clk,
        "e2e": e2e,
        # per step: the cold-start init + the iteration launches and work-list compactions of run()
        "gpu_launches": args.steps * (1 + eng.launches_per_run(n_iter)),
    }
    if args.config == "c1" and rank == 0:
        # second headline of the metric: ms per converged solve (C1, SingleParams() defaults,
        # 261 AM iterations) through the drop-in public API, host numpy in / out
        from paper_2408_10731_b200.solver_single import solve_single

        prob = scenarios.c1_problem()
        for _ in range(2):
            solve_single(prob, SingleParams())
        reps = 5
        t0 = time.perf_counter()
        for _ in range(reps):
            sol = solve_single(prob, SingleParams())
        ms = (time.perf_counter() - t0) / reps * 1e3
        from oracle import alg1 as O

        tr = np.stack([o.centers for o in prob.obstacles])
        op = O.Problem(P=prob.basis.P, Pd=prob.basis.Pdot, Pdd=prob.basis.Pddot,
                       bvals=np.stack([bc.values() for bc in prob.boundary])[None], desired=prob.desired[None],
                       tracks=tr, a=np.array([o.shape.a for o in prob.obstacles]),
                       b=np.array([o.shape.b for o in prob.obstacles]))
        t0 = time.perf_counter()
        O.solve(op, O.Params())
        ref_ms = (time.perf_counter() - t0) * 1e3
        line["converged_solve"] = {"ms_per_solve": ms, "iterations": sol.iterations, "converged": sol.converged,
                                   "api": "solver_single.solve_single (host numpy in/out, wall clock)",
                                   "cpu_port_ms_per_solve": ref_ms}
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        # bounded sample: ~40 member-solves per host core (C5 ~0.45 s each -> ~20 s of CPU work)
        sample = 40 * (os.cpu_count() or 1) if args.config != "c1" else 2 * (os.cpu_count() or 1)
        v, info = cpu_reference(args.config, sample)
        line["cpu_baseline"] = {"value": v, "unit": "traj-it/s", "cores": info["cores"], "kind": "port", "cpu_model": _cpu_model(),
                                "sample": f"{sample} members x {info['iterations']} AM its of the same recipe, "
                                          f"oracle port of solver_single (1 BLAS thread/process), "
                                          f"wall {info['wall_s']:.1f}s"}
    if rank == 0:
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()


def run_reference(args):
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    if args.config == "c3":
        vals = []
        for k in range(args.warmup + args.steps):
            v, info = cpu_reference_c3()
            if k >= args.warmup:
                vals.append(v)
        value = statistics.mean(vals)
        print(json.dumps({"impl": "reference", "metric": "problem-iterations/sec (joint 16-agent problems x iterations)",
                          "value": value, "unit": "problem-it/s", "n_gpus": world, "steps": args.steps,
                          "warmup": args.warmup, "higher_is_better": True, "scaling": "strong", "vs_baseline": None,
                          "dtype": "f64", "data": "synthetic", "config": {"workload": CONFIGS["c3"][3]},
                          "cpu_baseline": {"value": value, "unit": "problem-it/s", "cores": info["cores"],
                                           "kind": "port", "cpu_model": _cpu_model(), "sample": info["sample"]},
                          "e2e": {"value": value, "unit": "problem-it/s", "h2d_bytes_per_step": 0,
                                  "d2h_bytes_per_step": 0}}), flush=True)
        return
    if args.config == "c2alt":
        vals = []
        for k in range(args.warmup + args.steps):
            v, info = cpu_reference_c2alt()
            if k >= args.warmup:
                vals.append(v)
        value = statistics.mean(vals)
        print(json.dumps({"impl": "reference", "metric": "trajectory-iterations/sec (Alg. 2 batch x iterations)",
                          "value": value, "unit": "traj-it/s", "n_gpus": world, "steps": args.steps,
                          "warmup": args.warmup, "higher_is_better": True, "scaling": "strong", "vs_baseline": None,
                          "dtype": "f64", "data": "synthetic", "config": {"workload": CONFIGS["c2alt"][3]},
                          "cpu_baseline": {"value": value, "unit": "traj-it/s", "cores": info["cores"],
                                           "kind": "port", "cpu_model": _cpu_model(), "sample": info["sample"]},
                          "e2e": {"value": value, "unit": "traj-it/s", "h2d_bytes_per_step": 0,
                                  "d2h_bytes_per_step": 0}}), flush=True)
        return
    if args.config in ("mpc", "val"):
        vals = []
        for k in range(args.warmup + args.steps):
            if args.config == "mpc":
                v, info = cpu_reference_mpc()
                unit, metric = "robot-steps/s", "robot control steps/sec (receding horizon, 40 warm AM its per step)"
            else:
                v, info = cpu_reference_val()
                unit, metric = "traj/s", "trajectories validated/sec (raw-geometry metrics + collision check)"
            if k >= args.warmup:
                vals.append(v)
        value = statistics.mean(vals)
        print(json.dumps({"impl": "reference", "metric": metric, "value": value, "unit": unit, "n_gpus": world,
                          "steps": args.steps, "warmup": args.warmup, "higher_is_better": True, "scaling": "strong",
                          "vs_baseline": None, "dtype": "f64", "data": "synthetic",
                          "config": {"workload": CONFIGS[args.config][3]},
                          "cpu_baseline": {"value": value, "unit": unit, "cores": 1, "kind": "port", "cpu_model": _cpu_model(), "sample": info},
                          "e2e": {"value": value, "unit": unit, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}),
              flush=True)
        return
    if args.config == "c4":
        vals = []
        for k in range(args.warmup + args.steps):
            v, info = cpu_reference_c4()
            if k >= args.warmup:
                vals.append(v)
        value = statistics.mean(vals)
        print(json.dumps({"impl": "reference", "metric": "sample-inner-iterations/sec (PRIEST projection, CEM rounds)",
                          "value": value, "unit": "sample-inner-it/s", "n_gpus": world, "steps": args.steps,
                          "warmup": args.warmup, "higher_is_better": True, "scaling": "strong", "vs_baseline": None,
                          "dtype": "f64", "data": "synthetic", "config": {"workload": CONFIGS["c4"][3]},
                          "cpu_baseline": {"value": value, "unit": "sample-inner-it/s", "cores": info["cores"],
                                           "kind": "port", "cpu_model": _cpu_model(), "sample": info["sample"]},
                          "e2e": {"value": value, "unit": "sample-inner-it/s", "h2d_bytes_per_step": 0,
                                  "d2h_bytes_per_step": 0}}), flush=True)
        return
    n_o, members_total, n_iter, desc = CONFIGS[args.config]
    procs = os.cpu_count() or 1
    sample = procs if args.config != "c1" else 1
    vals = []
    info = None
    for k in range(args.warmup + args.steps):
        v, info = cpu_reference(args.config, sample, procs)
        if k >= args.warmup:
            vals.append(v)
    value = statistics.mean(vals)
    line = {
        "impl": "reference",
        "metric": "trajectory-iterations/sec (batch x AM iters)",
        "value": value,
        "unit": "traj-it/s",
        "n_gpus": world,
        "steps": args.steps,
        "warmup": args.warmup,
        "ms_per_step": info["wall_s"] * 1e3,
        "higher_is_better": True,
        "scaling": "strong",
        "vs_baseline": None,
        "dtype": "f64",
        "data": "synthetic (seeded scenario recipe, SURVEY.md §8(d))",
        "config": {"workload": desc, "members": members_total, "n_obs": n_o, "n_p": 100, "am_iters": n_iter},
        "cpu_baseline": {"value": value, "unit": "traj-it/s", "cores": procs, "kind": "port", "cpu_model": _cpu_model(),
                         "sample": f"{sample} members x {n_iter} AM its per step (bounded sample of the workload)"},
        "e2e": {"value": value, "unit": "traj-it/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


def _free_port() -> int:
    import socket

    with socket.socket(socket.AF_INET, socket.SOCK_STREAM) as sk:
        sk.bind(("127.0.0.1", 0))
        return int(sk.getsockname()[1])


def _spawn_ranks(n: int) -> int:
    """`bench.py --gpus N` without a launcher: re-run this command under torch.distributed.run with one rank
    per GPU (NCCL over NVLink; rendezvous on 127.0.0.1) and return its exit code."""
    env = dict(os.environ)
    env.setdefault("NCCL_DEBUG", "INFO")  # the NCCL init lines (transport, NVLS) land on stderr
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={n}",
           "--master-addr=127.0.0.1", f"--master-port={_free_port()}", os.path.abspath(__file__)] + sys.argv[1:]
    return subprocess.call(cmd, env=env)


def main():
    args = parse()
    world = int(os.environ.get("WORLD_SIZE", "0"))
    if args.gpus > 1 and world == 0:
        raise SystemExit(_spawn_ranks(args.gpus))
    if world and world != args.gpus:
        raise SystemExit(f"bench: --gpus {args.gpus} but the launcher started {world} ranks")
    if args.impl == "reference":
        run_reference(args)
    elif args.config == "c4":
        run_c4(args)
    elif args.config == "c3":
        run_c3(args)
    elif args.config == "c2alt":
        run_c2alt(args)
    elif args.config == "val":
        run_val(args)
    elif args.config == "mpc":
        run_mpc(args)
    else:
        run_b200(args)


if __name__ == "__main__":
    main()
