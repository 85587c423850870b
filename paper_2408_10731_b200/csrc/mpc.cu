// Scenario-to-device adapters and the receding-horizon fleet step, sm_100a.
//
// predict_tracks_kernel: constant-velocity obstacle extrapolation (bench/scenarios.py:118-127) for S
//   scenarios / prediction times in one launch, element-parallel, in numpy's operation order with
//   explicitly rounded intrinsics (no FMA contraction), so the tracks are bit-identical to the host's.
// mpc_advance_kernel: the per-control-step bookkeeping of bench/runner.py:362-428 for B robots at once, one
//   CTA per robot, between two solves of a device-resident Alg. 1 engine: execute the first n_exec samples
//   of the plan against the TRUE obstacle motion, freeze robots that collided or reached the goal, and
//   write the next problem (boundary, desired line, q) plus the warm-start d, so no state leaves the GPU.
#include "common.cuh"
#include "fastmath.cuh"
#include "alg1_elem.cuh"
#include "../../include/trajopt_b200.h"

namespace tro {

__global__ void predict_tracks_kernel(tro_track_dims d, const double* __restrict__ c, const double* __restrict__ v,
                                      const double* __restrict__ t, const double* __restrict__ t_now,
                                      double* __restrict__ out) {
    const int n_p = d.n_p, n_o = d.n_obs, dim = d.dim;
    const int64_t total = (int64_t)d.n_scen * n_o * n_p;
    const double t0 = __ldg(t);
    for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < total;
         e += (int64_t)gridDim.x * blockDim.x) {
        const int k = (int)(e % n_p);
        const int64_t sj = e / n_p;  // scenario * n_o + obstacle
        const int s = (int)(sj / n_o);
        // (t_now + t) - t[0], then v * rel, then c + (v * rel): numpy's order, each step rounded once
        const double rel = __dsub_rn(__dadd_rn(__ldg(t_now + s), __ldg(t + k)), t0);
        const int64_t ob = (d.shared_obstacles ? sj % n_o : sj) * dim;
        for (int ax = 0; ax < dim; ++ax) {
            const double val = __dadd_rn(__ldg(c + ob + ax), __dmul_rn(__ldg(v + ob + ax), rel));
            if (d.layout)
                out[(sj * dim + ax) * n_p + k] = val;  // engine layout: a word's samples contiguous
            else
                out[(sj * n_p + k) * dim + ax] = val;
        }
    }
}

constexpr int kMpcThreads = 128;
constexpr int kMpcMaxExec = 64;

struct MpcArgs {
    tro_mpc_dims d;
    tro_mpc_consts c;
    tro_alg1_state e;
    tro_mpc_io io;
};

// runner.py:314-323 _in_collision_now for ONE obstacle: raw shapes, centre c + v t, quad < 1
// (3-D: a, a, b; 2-D: a, b); every step rounded once in numpy's order
template <int DIM>
__device__ __forceinline__ bool hits(const MpcArgs& A, int j, const double* p, double t_abs) {
    const double a = __ldg(A.c.shape_a + j), b = __ldg(A.c.shape_b + j);
    const double a2 = __dmul_rn(a, a), b2 = __dmul_rn(b, b);
    double quad = 0.0;
#pragma unroll
    for (int ax = 0; ax < DIM; ++ax) {
        const double cen = __dadd_rn(__ldg(A.c.centers + j * DIM + ax),
                                     __dmul_rn(__ldg(A.c.velocities + j * DIM + ax), t_abs));
        const double dl = __dsub_rn(p[ax], cen);
        const double term = __ddiv_rn(__dmul_rn(dl, dl), ax == DIM - 1 ? b2 : a2);
        quad = ax == 0 ? term : __dadd_rn(quad, term);
    }
    return quad < 1.0;
}

// every (sample, obstacle) pair of the CTA's samples in parallel; bit s of the result: sample s collides
template <int DIM>
__device__ unsigned long long collide_mask(const MpcArgs& A, const double* pts, int stride, const double* times,
                                           int n_s, unsigned long long* sMask) {
    const int tid = threadIdx.x;
    if (tid == 0) *sMask = 0ull;
    __syncthreads();
    unsigned long long mine = 0ull;
    for (int o = tid; o < n_s * A.d.n_obs; o += kMpcThreads) {
        const int smp = o / A.d.n_obs, j = o - smp * A.d.n_obs;
        if (hits<DIM>(A, j, pts + smp * stride, times[smp])) mine |= 1ull << smp;
    }
    if (mine) atomicOr(sMask, mine);
    __syncthreads();
    return *sMask;
}

template <int DIM, int MODE>
__global__ void __launch_bounds__(kMpcThreads) mpc_advance_kernel(MpcArgs A) {
    extern __shared__ double sm[];
    __shared__ double sNew[3 * DIM];  // executed state: pos, vel, acc
    __shared__ int sFlag;
    const int i = blockIdx.x, tid = threadIdx.x;
    const int n_p = A.d.n_p, m = A.d.m, n_o = A.d.n_obs, n_exec = A.d.n_exec;
    double* sXi = sm;                    // DIM x m
    double* sEx = sXi + DIM * m;         // n_exec x (pos, vel, acc) x DIM
    double* sDes = sEx + n_exec * 3 * DIM;  // n_p x DIM
    const double* goal = A.c.goal + (int64_t)i * DIM;
    double* bv = A.io.bvals + (int64_t)i * DIM * 6;

    if constexpr (MODE == 1) {
        if (A.io.flags[i]) return;  // frozen: status stays TRO_CONVERGED, nothing is recorded
        if (tid == 0 && A.io.res_out) A.io.res_out[i] = A.e.res_norm[i];
        // warm d of the final iterate (d_step's line-of-sight scale of the last positions against this
        // step's planning tracks) for the next solve's first iteration; same expression as the engine
        if (A.io.d) {
            const double* pos = A.e.pos + (int64_t)i * DIM * n_p;
            double* dd = A.io.d + (int64_t)i * n_o * n_p;
            for (int e = tid; e < n_o * n_p; e += kMpcThreads) {
                const int j = e / n_p, t = e - j * n_p;
                const double pa = __ldg(A.c.plan_a + j), pb = __ldg(A.c.plan_b + j);
                const double ia2 = 1.0 / (pa * pa), ib2 = 1.0 / (pb * pb);
                const double* tr = A.c.tracks + (int64_t)j * DIM * n_p + t;
                const double ex = pos[t] - __ldg(tr), ey = pos[n_p + t] - __ldg(tr + n_p);
                double qd;
                if constexpr (DIM == 3) {
                    const double ez = pos[2 * n_p + t] - __ldg(tr + 2 * n_p);
                    qd = ex * ex * ia2 + ey * ey * ia2 + ez * ez * ib2;
                } else {
                    qd = ex * ex * ia2 + ey * ey * ib2;
                }
                dd[e] = los_scale(qd);
            }
        }
        for (int k = tid; k < DIM * m; k += kMpcThreads) sXi[k] = A.e.xi[(int64_t)i * DIM * m + k];
        __syncthreads();
        // traj.pos / vel / acc rows 1..n_exec of the plan (runner.py:407-410)
        for (int o = tid; o < n_exec * 3 * DIM; o += kMpcThreads) {
            const int s = o / (3 * DIM), r = o - s * 3 * DIM, kind = r / DIM, ax = r - kind * DIM;
            const double* row = (kind == 0 ? A.c.P : kind == 1 ? A.c.Pdot : A.c.Pddot) + (int64_t)(s + 1) * m;
            double acc = 0.0;
            for (int cc = 0; cc < m; ++cc) acc = fma(__ldg(row + cc), sXi[ax * m + cc], acc);
            sEx[o] = acc;
        }
        __syncthreads();
        __shared__ double sT[kMpcMaxExec];
        __shared__ unsigned long long sMask;
        for (int k = tid; k < n_exec; k += kMpcThreads) sT[k] = __ldg(A.c.t_exec + k);
        __syncthreads();
        const unsigned long long coll = collide_mask<DIM>(A, sEx, 3 * DIM, sT, n_exec, &sMask);
        if (tid == 0) {
            // runner.py:407-419, in order per sample: append, collision at its time, then goal proximity
            int nt = A.io.n_trace[i], fl = 0, stop = n_exec - 1;
            double* tr = A.io.trace + (int64_t)i * A.d.trace_cap * DIM;
            for (int s = 0; s < n_exec; ++s) {
                const double* p = sEx + s * 3 * DIM;
                if (nt < A.d.trace_cap) {
#pragma unroll
                    for (int ax = 0; ax < DIM; ++ax) tr[nt * DIM + ax] = p[ax];
                }
                ++nt;
                if ((coll >> s) & 1ull) {
                    fl = 1;
                    stop = s;
                    break;
                }
                double g2 = 0.0;
#pragma unroll
                for (int ax = 0; ax < DIM; ++ax) {
                    const double e = __dsub_rn(p[ax], goal[ax]);
                    g2 = __dadd_rn(g2, __dmul_rn(e, e));
                }
                if (__dsqrt_rn(g2) <= A.c.goal_radius) {
                    fl = 2;
                    stop = s;
                    break;
                }
            }
            A.io.n_trace[i] = nt;
            A.io.flags[i] = fl;
            sFlag = fl;
#pragma unroll
            for (int k = 0; k < 3 * DIM; ++k) sNew[k] = sEx[stop * 3 * DIM + k];
        }
    } else {
        // episode start (runner.py:349-358): the robot at rest at the boundary's start
        __shared__ unsigned long long sMask;
        __shared__ double sStart[DIM];
        const double t0 = 0.0;
        if (tid < DIM) {
            sStart[tid] = bv[tid * 6 + 0];
            sNew[tid] = sStart[tid];
            sNew[DIM + tid] = 0.0;
            sNew[2 * DIM + tid] = 0.0;
            A.io.trace[(int64_t)i * A.d.trace_cap * DIM + tid] = sStart[tid];
        }
        __syncthreads();
        const unsigned long long coll = collide_mask<DIM>(A, sStart, DIM, &t0, 1, &sMask);
        if (tid == 0) {
            A.io.n_trace[i] = 1;
            const int fl = (coll & 1ull) ? 1 : 0;
            A.io.flags[i] = fl;
            sFlag = fl;
        }
    }
    __syncthreads();
    if (sFlag) {
        if (tid == 0) A.e.status[i] = TRO_CONVERGED;  // frozen for the rest of the episode
        return;
    }
    // next problem (runner.py:365-375): boundary = executed state, desired = pos + frac (goal - pos)
    if (tid < DIM) {
        const int ax = tid;
        bv[ax * 6 + 0] = sNew[ax];
        bv[ax * 6 + 1] = sNew[DIM + ax];
        bv[ax * 6 + 2] = sNew[2 * DIM + ax];
        bv[ax * 6 + 3] = goal[ax];
        bv[ax * 6 + 4] = 0.0;
        bv[ax * 6 + 5] = 0.0;
    }
    double* dg = A.io.desired + (int64_t)i * n_p * DIM;
    for (int o = tid; o < n_p * DIM; o += kMpcThreads) {
        const int t = o / DIM, ax = o - t * DIM;
        const double p = sNew[ax];
        const double v = __dadd_rn(p, __dmul_rn(__ldg(A.c.frac + t), __dsub_rn(goal[ax], p)));
        sDes[o] = v;
        dg[o] = v;
    }
    __syncthreads();
    // q = -2 w_track (P' desired)' (solver_single.py:173): a warp per output, lanes over samples
    const double w2 = -2.0 * A.c.w_track;
    const int warp = tid >> 5, lane = tid & 31;
    for (int o = warp; o < DIM * m; o += kMpcThreads / 32) {
        const int ax = o / m, cc = o - ax * m;
        double s = 0.0;
        for (int t = lane; t < n_p; t += 32) s = fma(__ldg(A.c.P + (int64_t)t * m + cc), sDes[t * DIM + ax], s);
        s = warp_sum(s);
        if (lane == 0) A.io.q[(int64_t)i * DIM * m + o] = w2 * s;
    }
    // a fresh solve_single call on the warm state: iteration = 0 (runner.py:376-377), solve-local history
    if (tid == 0) {
        A.e.status[i] = 0;
        A.e.iteration[i] = 0;
        A.e.last_change[i] = 0;
        A.e.n_hist[i] = 0;
        A.e.n_changes[i] = 0;
    }
    for (int k = tid; k < A.d.ring_len; k += kMpcThreads) A.e.ring[(int64_t)i * A.d.ring_len + k] = 0.0;
}

}  // namespace tro

extern "C" int tro_predict_tracks_f64(const tro_track_dims* d, const double* centers, const double* velocities,
                                      const double* t, const double* t_now, double* out, void* stream) {
    if (!d || d->n_scen < 0 || d->n_obs < 0 || d->n_p < 1 || (d->dim != 2 && d->dim != 3)) return TRO_EINVAL;
    const int64_t total = (int64_t)d->n_scen * d->n_obs * d->n_p;
    if (total == 0) return 0;
    if (!centers || !velocities || !t || !t_now || !out) return TRO_EINVAL;
    const int threads = 256;
    const int64_t want = (total + threads - 1) / threads;
    const unsigned blocks = (unsigned)(want < 148 * 16 ? want : 148 * 16);
    tro::predict_tracks_kernel<<<blocks, threads, 0, reinterpret_cast<cudaStream_t>(stream)>>>(*d, centers, velocities,
                                                                                                  t, t_now, out);
    return (int)cudaGetLastError();
}

extern "C" int tro_mpc_advance_f64(int32_t mode, const tro_mpc_dims* d, const tro_mpc_consts* c,
                                   const tro_alg1_state* e, const tro_mpc_io* io, void* stream) {
    if (!d || !c || !e || !io || (mode != 0 && mode != 1) || (d->dim != 2 && d->dim != 3) || d->n_p < 2 ||
        d->m < 1 || d->n_obs < 0 || d->n_exec < 1 || d->n_exec > tro::kMpcMaxExec || d->n_exec >= d->n_p ||
        d->trace_cap < 1 || d->ring_len < 0)
        return TRO_EINVAL;
    if (!c->P || !c->frac || !c->goal || !io->bvals || !io->q || !io->desired || !io->trace || !io->n_trace ||
        !io->flags || !e->status || !e->iteration || !e->last_change || !e->n_hist || !e->n_changes)
        return TRO_EINVAL;
    if (d->n_obs > 0 && (!c->centers || !c->velocities || !c->shape_a || !c->shape_b)) return TRO_EINVAL;
    if (mode == 1 && (!c->Pdot || !c->Pddot || !c->t_exec || !e->xi || !e->res_norm ||
                      (io->d && (!e->pos || !c->tracks || !c->plan_a || !c->plan_b))))
        return TRO_EINVAL;
    if (d->n_members <= 0) return 0;
    tro::MpcArgs A;
    A.d = *d;
    A.c = *c;
    A.e = *e;
    A.io = *io;
    const size_t smem = sizeof(double) * ((size_t)d->dim * d->m + (size_t)d->n_exec * 3 * d->dim +
                                          (size_t)d->n_p * d->dim);
    if (smem > 200 * 1024) return TRO_EINVAL;
    cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
    const unsigned blocks = (unsigned)d->n_members;
#define TRO_MPC_LAUNCH(D, M)                                                                                 \
    do {                                                                                                     \
        cudaFuncSetAttribute(tro::mpc_advance_kernel<D, M>, cudaFuncAttributeMaxDynamicSharedMemorySize,   \
                             (int)smem);                                                                     \
        tro::mpc_advance_kernel<D, M><<<blocks, tro::kMpcThreads, smem, st>>>(A);                            \
    } while (0)
    if (d->dim == 3) {
        if (mode) TRO_MPC_LAUNCH(3, 1); else TRO_MPC_LAUNCH(3, 0);
    } else {
        if (mode) TRO_MPC_LAUNCH(2, 1); else TRO_MPC_LAUNCH(2, 0);
    }
#undef TRO_MPC_LAUNCH
    return (int)cudaGetLastError();
}

namespace tro {
// order[] = indices with flags == 0, increasing (a single CTA: block-wide exclusive scan per 1024-chunk)
__global__ void __launch_bounds__(1024) mpc_compact_kernel(int n, const int32_t* __restrict__ flags,
                                                            int32_t* __restrict__ order, int32_t* n_order) {
    __shared__ int sWarpSum[32];
    __shared__ int sBase;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    if (tid == 0) sBase = 0;
    __syncthreads();
    for (int c0 = 0; c0 < n; c0 += 1024) {
        const int k = c0 + tid;
        const int keep = (k < n && __ldg(flags + k) == 0) ? 1 : 0;
        const unsigned ball = __ballot_sync(0xffffffffu, keep);
        const int before = __popc(ball & ((1u << lane) - 1u));
        if (lane == 0) sWarpSum[warp] = __popc(ball);
        __syncthreads();
        int wbase = 0;
        for (int w = 0; w < warp; ++w) wbase += sWarpSum[w];
        if (keep) order[sBase + wbase + before] = k;
        __syncthreads();
        if (tid == 0) {
            int tot = 0;
            for (int w = 0; w < 32; ++w) tot += sWarpSum[w];
            sBase += tot;
        }
        __syncthreads();
    }
    if (tid == 0) *n_order = sBase;
}
}  // namespace tro

extern "C" int tro_mpc_compact(int32_t n_members, const int32_t* flags, int32_t* order, int32_t* n_order,
                               void* stream) {
    if (n_members < 0 || !n_order || (n_members > 0 && (!flags || !order))) return TRO_EINVAL;
    tro::mpc_compact_kernel<<<1, 1024, 0, reinterpret_cast<cudaStream_t>(stream)>>>(n_members, flags, order,
                                                                                     n_order);
    return (int)cudaGetLastError();
}
