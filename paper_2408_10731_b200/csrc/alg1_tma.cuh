// Persistent, warp-specialised fused AM iteration (Alg. 1) for sm_100a.
//
// Three warp roles per CTA:
//   * a PRODUCER warp (one elected lane) streams each member's obstacle rows of state into a shared-memory
//     ring with TMA bulk copies (cp.async.bulk ... mbarrier::complete_tx).  In the interleaved layout
//     state[i][j][w][t] the W words x NP samples of one obstacle row are ONE contiguous block (fp64 3-D:
//     7200 B), so a stage (G rows) is one bulk copy (plus one for the track rows when the obstacles are
//     not constant-velocity tracks the kernel can generate itself);
//   * CONSUMER warps (G*NP threads: sample t, obstacle group g) run the element pass out of the ring and
//     write the new state straight back to HBM;
//   * a SCALAR warp runs each member's QP prologue (q_lin, xi = K^-1 [-q_lin; b], positions) and epilogue
//     (fixed-order obstacle sums, residual norm / max, history, stall rule) OFF the consumers' path: the
//     prologue of the next member and the epilogue of the previous one run while the consumers stream
//     the current member.  Positions, reduction partials and the member's penalties are double-buffered
//     in shared memory (buffer = active-unit count & 1) and handed over with mbarriers
//     (ready[b]: scalar -> consumers, done[b]: consumers -> scalar).
// Measured (tools/ab_alg1_exp.sh): taking the prologue off the consumers' path alone moved the C5 launch
// from 0.78 to 0.85 of HBM.
//
// Grid = min(B, SMs * MINB): each CTA walks members i = blockIdx.x, += gridDim.x (or the work list).
#pragma once
#include "alg1_elem.cuh"
#include "tma.cuh"

namespace tro {

template <int DIM, typename T, int LAY, int NP, int G>
struct TmaCfg {
    static constexpr int W = Words<DIM, LAY>::W;
    static constexpr int kRowBytes = W * NP * (int)sizeof(T);  // one obstacle row of state
    static constexpr int kTrkBytes = DIM * NP * 8;             // one obstacle row of tracks
    static constexpr int kConsumers = ((G * NP + 31) / 32) * 32;
    static constexpr int kThreads = kConsumers + 64;           // + scalar warp + producer warp
    static_assert(kRowBytes % 16 == 0 && kTrkBytes % 16 == 0, "bulk copies need 16-byte rows");
};

constexpr int kTmaMaxStages = 8;

// shared-memory carve-up (bytes), buffers [2] are double-buffered per active unit:
// [stages | P | pos_prev[2] | pos_new[2] | sums_in | red[2] | shapes | lin | qlin | xi[2] | warp[2] | scal[2] | bars]
struct TmaLayout {
    int stages, stage_bytes, n_stages, P, pos_prev, pos_new, sums_in, red, shp, lin, shpT, linT, trks, qlin, xi, warp,
        scal, kmat, qb, sched, bars, total;
};
__host__ __device__ inline TmaLayout tma_layout(int row_bytes, int trk_bytes, bool lin, int n_stages, int n_p, int m,
                                                int dim, int n_o, int G, int consumers) {
    TmaLayout L;
    L.stage_bytes = G * (row_bytes + (lin ? 0 : trk_bytes));
    L.n_stages = n_stages;
    int off = 0;
    L.stages = off;   off += n_stages * L.stage_bytes;
    L.P = off;        off += n_p * m * 8;
    L.pos_prev = off; off += 2 * dim * n_p * 8;
    L.pos_new = off;  off += 2 * dim * n_p * 8;
    L.sums_in = off;  off += 2 * dim * n_p * 8;
    L.red = off;      off += 2 * G * 2 * dim * n_p * 8;
    off = (off + 15) & ~15;
    L.shp = off;      off += 4 * (n_o > 0 ? n_o : 1) * 8;  // per obstacle {a, b, 1/a^2, 1/b^2} (two 16-B loads)
    L.lin = off;      off += lin ? (6 * (n_o > 0 ? n_o : 1) + n_p) * 8 : 0;  // {c, v} per obstacle + rel times
    L.shpT = off;     off += 4 * (n_o > 0 ? n_o : 1) * 4;  // fp32 builds: the shape records in float
    off = (off + 15) & ~15;
    L.linT = off;     off += lin ? (6 * (n_o > 0 ? n_o : 1) + n_p) * 4 : 0;  // fp32 builds: the track records
    off = (off + 15) & ~15;
    L.trks = off;     off += dim * n_p * 8;  // sum over obstacles of the track centres per (axis, sample)
    L.qlin = off;     off += dim * 16 * 8;
    L.xi = off;       off += 2 * dim * 16 * 8;
    L.warp = off;     off += 2 * 2 * (consumers / 32) * 8;
    L.scal = off;     off += 2 * 2 * 8;
    L.kmat = off;     off += kMaxNk * kMaxNk * 8;        // the member's K^-1 level (scalar warp)
    L.qb = off;       off += dim * (16 + kMaxNk) * 8;    // the member's q and boundary values (scalar warp)
    off = (off + 15) & ~15;
    L.sched = off;    off += 2 * (int)((sizeof(SchedS) + 15) & ~(size_t)15);  // [2] bookkeeping mirrors
    off = (off + 15) & ~15;
    L.bars = off;     off += (2 * kTmaMaxStages + 4) * 8;
    L.total = off;
    return L;
}

// Work unit u of this CTA: a member and the stage range [st0, st1) of its obstacle rows (half: -1 = whole
// member, 0 / 1 = the first / second half of a tail member)
struct WorkUnit {
    int pos, member, st0, st1, half;  // pos: index into the work list (order, or the members themselves)
};
__device__ __forceinline__ WorkUnit work_unit(int u, int rounds, int split_tail, int nst, const int32_t* order) {
    WorkUnit w;
    if (split_tail && u == rounds) {
        const int h = (int)blockIdx.x & 1, mid = nst / 2;
        w.pos = rounds * (int)gridDim.x + (int)blockIdx.x / 2;
        w.st0 = h ? mid : 0;
        w.st1 = h ? nst : mid;
        w.half = h;
    } else {
        w.pos = (int)blockIdx.x + u * (int)gridDim.x;
        w.st0 = 0;
        w.st1 = nst;
        w.half = -1;
    }
    w.member = order ? __ldg(order + w.pos) : w.pos;
    return w;
}

// The next unit >= u that is active (not frozen, level passes the cond guard); n_units if none.  Every role
// walks the same sequence: a member's status and level are only written by its own epilogue, after every
// role has passed it.
__device__ __forceinline__ int next_active(const Alg1Args& A, int u, int n_units, int rounds, int split_tail, int nst,
                                           const int32_t* order, WorkUnit* wu) {
    for (; u < n_units; ++u) {
        *wu = work_unit(u, rounds, split_tail, nst, order);
        const int st = A.s.status[wu->member];
        if (!(st & (TRO_CONVERGED | TRO_FACTOR_FAILED)) && A.c.level_ok[A.s.level[wu->member]]) return u;
    }
    return n_units;
}

// DM: the previous iterate's d source fixed at compile time (2: recompute, the steady state) or -1 (read
// A.p.d_mode at run time: the first iteration after an init / prime).  EXP: the optional d / copies exports
// exist (false: compiled out, the steady state of the benchmarks)
template <int DIM, typename T, int LAY, int NP, int G, int MINB, int DM, bool EXP = true>
__global__ void __launch_bounds__(TmaCfg<DIM, T, LAY, NP, G>::kThreads, MINB) alg1_tma_kernel(Alg1Args A) {
    using C = TmaCfg<DIM, T, LAY, NP, G>;
    constexpr int W = C::W;
    constexpr int NC = C::kConsumers;
    constexpr int NCW = NC / 32;
    extern __shared__ __align__(128) unsigned char smraw[];
    const int n_o = A.d.n_obs, m = A.d.m, ne = A.d.n_eq, nk = m + ne;
    const int B = A.d.n_members;
    const bool lin = A.c.track_lin != nullptr;
    const int S = A.n_stages;
    const TmaLayout L = tma_layout(C::kRowBytes, C::kTrkBytes, lin, S, NP, m, DIM, n_o, G, NC);
    unsigned char* stages = smraw + L.stages;
    double* sP = reinterpret_cast<double*>(smraw + L.P);
    double* sPosPrev = reinterpret_cast<double*>(smraw + L.pos_prev);  // [2][DIM * NP]
    double* sPosNew = reinterpret_cast<double*>(smraw + L.pos_new);    // [2][DIM * NP]
    double* sSumIn = reinterpret_cast<double*>(smraw + L.sums_in);
    double* sRed = reinterpret_cast<double*>(smraw + L.red);           // [2][G * 2 * DIM * NP]
    double* sShp = reinterpret_cast<double*>(smraw + L.shp);
    double* sLin = reinterpret_cast<double*>(smraw + L.lin);
    float* sShpF = reinterpret_cast<float*>(smraw + L.shpT);
    float* sLinF = reinterpret_cast<float*>(smraw + L.linT);
    double* sTrk = reinterpret_cast<double*>(smraw + L.trks);  // [DIM * NP]
    double* sQlin = reinterpret_cast<double*>(smraw + L.qlin);
    double* sXi = reinterpret_cast<double*>(smraw + L.xi);             // [2][DIM * 16]
    double* sWarp = reinterpret_cast<double*>(smraw + L.warp);         // [2][2 * NCW]
    double* sScal = reinterpret_cast<double*>(smraw + L.scal);         // [2][rho, rho_o]
    double* sK = reinterpret_cast<double*>(smraw + L.kmat);
    double* sQ = reinterpret_cast<double*>(smraw + L.qb);              // [DIM * 16] q, then [DIM * ne] bvals
    double* sBv = sQ + DIM * 16;
    constexpr int kSchedBytes = (int)((sizeof(SchedS) + 15) & ~(size_t)15);
    SchedS* sSched = reinterpret_cast<SchedS*>(smraw + L.sched);       // [2] (stride kSchedBytes)
    uint64_t* full = reinterpret_cast<uint64_t*>(smraw + L.bars);
    uint64_t* empty = full + kTmaMaxStages;
    uint64_t* ready = empty + kTmaMaxStages;  // [2] scalar warp -> consumers: prologue of the unit in buffer b
    uint64_t* done = ready + 2;               // [2] consumers -> scalar warp: partials of buffer b written
    constexpr int kRedBuf = G * 2 * DIM * NP;

    const int tid = threadIdx.x;
    const int warp = tid >> 5, lane = tid & 31;

    // ---------------- one-time setup: barriers, basis, shapes, linear tracks
    if (tid == 0) {
        for (int s = 0; s < S; ++s) {
            mbar_init(&full[s], 1);
            mbar_init(&empty[s], NCW);
        }
        for (int b = 0; b < 2; ++b) {
            mbar_init(&ready[b], 1);
            mbar_init(&done[b], NCW);
        }
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    for (int k = tid; k < NP * m; k += blockDim.x) sP[k] = ld_const(A.c.P + k);
    for (int k = tid; k < n_o; k += blockDim.x) {
        const double a = ld_const(A.c.shape_a + k), b = ld_const(A.c.shape_b + k);
        sShp[4 * k + 0] = a;
        sShp[4 * k + 1] = b;
        sShp[4 * k + 2] = 1.0 / (a * a);
        sShp[4 * k + 3] = 1.0 / (b * b);
    }
    if (lin)
        for (int k = tid; k < 6 * n_o + NP; k += blockDim.x) sLin[k] = ld_const(A.c.track_lin + k);
    if constexpr (sizeof(T) == 4) {
        for (int k = tid; k < 4 * n_o; k += blockDim.x) {
            const double a = ld_const(A.c.shape_a + k / 4), b = ld_const(A.c.shape_b + k / 4);
            const int c = k & 3;
            sShpF[k] = (float)(c == 0 ? a : c == 1 ? b : c == 2 ? 1.0 / (a * a) : 1.0 / (b * b));
        }
        if (lin)
            for (int k = tid; k < 6 * n_o + NP; k += blockDim.x) sLinF[k] = (float)ld_const(A.c.track_lin + k);
    }
    __syncthreads();  // sLin complete
    // the obstacle-summed track centres of every sample: the target sums the next position step needs are
    // sum_j (centre_j + offset_j); the consumers accumulate only the offsets and the epilogue adds these
    for (int k = tid; k < DIM * NP; k += blockDim.x) {
        const int ax = k / NP, tt = k - ax * NP;
        double acc = 0.0;
        if (lin) {
            const double rel = sLin[6 * n_o + tt];
            for (int j = 0; j < n_o; ++j)
                acc += __dadd_rn(sLin[6 * j + ax], __dmul_rn(sLin[6 * j + DIM + ax], rel));
        } else {
            for (int j = 0; j < n_o; ++j) acc += ld_const(A.c.tracks + ((int64_t)j * DIM + ax) * NP + tt);
        }
        sTrk[k] = acc;
    }
    __syncthreads();

    const int nst = (n_o + G - 1) / G;  // stages per member
    // the work list: order[0 .. *n_order) when given (e.g. the robots still driving), else members 0..B-1;
    // `rounds` full rounds and then, with tail balancing, one half (of the stages) of a tail member for
    // the first 2 * tail CTAs
    const int32_t* order = A.s.order;
    const int n_work = order ? *A.s.n_order : B;
    const int rounds = n_work / (int)gridDim.x;
    const int tail = n_work - rounds * (int)gridDim.x;
    const int split_tail = (A.split_tail && tail > 0 && 2 * tail <= (int)gridDim.x) ? tail : 0;
    const int n_units = split_tail ? rounds + ((int)blockIdx.x < 2 * split_tail ? 1 : 0)
                                   : (n_work - (int)blockIdx.x + (int)gridDim.x - 1) / (int)gridDim.x;

    if (warp == NCW + 1) {
        // ======================= producer warp (one elected lane)
        if (lane == 0) {
            int s = 0;
            uint32_t ph = 0;
            bool wrapped = false;
            const int stage_tx = lin ? C::kRowBytes : C::kRowBytes + C::kTrkBytes;
            WorkUnit wu;
            for (int u = next_active(A, 0, n_units, rounds, split_tail, nst, order, &wu); u < n_units;
                 u = next_active(A, u + 1, n_units, rounds, split_tail, nst, order, &wu)) {
                const int i = wu.member;
                const unsigned char* src = reinterpret_cast<const unsigned char*>(A.s.state) +
                                           (int64_t)i * n_o * C::kRowBytes;
                const unsigned char* trk = reinterpret_cast<const unsigned char*>(A.c.tracks);
                for (int j0 = wu.st0 * G; j0 < n_o && j0 < wu.st1 * G; j0 += G) {
                    if (wrapped) mbar_wait(&empty[s], ph ^ 1u);  // the consumers released this stage
                    const int rows = min(G, n_o - j0);
                    unsigned char* buf = stages + s * L.stage_bytes;
                    mbar_expect_tx(&full[s], rows * stage_tx);
                    bulk_g2s(buf, src + (int64_t)j0 * C::kRowBytes, rows * C::kRowBytes, &full[s]);
                    if (!lin)
                        bulk_g2s(buf + G * C::kRowBytes, trk + (int64_t)j0 * C::kTrkBytes, rows * C::kTrkBytes,
                                 &full[s]);
                    if (++s == S) {
                        s = 0;
                        ph ^= 1u;
                        wrapped = true;
                    }
                }
            }
        }
        return;
    }

    if (warp == NCW) {
        // ======================= scalar warp: QP prologue / reduction epilogue, two units apart
        auto prologue = [&](const WorkUnit& wu, int b) {
            // Latency-conscious: a single warp does what 13 warps did, so every global read is issued up front
            // in unrolled batches (one memory latency per batch, not one per element), the K^-1 level, q and
            // the boundary values are staged in shared memory, and each lane owns whole dot products (no
            // shuffle chains).
            const int i = wu.member;
            const bool split = wu.half >= 0;
            constexpr int NPOS = DIM * NP, NSUM = 2 * DIM * NP;
            constexpr int RP = (NPOS + 31) / 32, RS = (NSUM + 31) / 32, RK = (kMaxNk * kMaxNk + 31) / 32;
            double* pPrev = sPosPrev + b * DIM * NP;
            double* pNew = sPosNew + b * DIM * NP;
            double* xs = sXi + b * DIM * 16;
            SchedS* S = reinterpret_cast<SchedS*>(reinterpret_cast<unsigned char*>(sSched) + b * kSchedBytes);
            const int level = A.s.level[i];  // broadcast; the K^-1 rows below depend on it
            const double* posg = A.s.pos + (int64_t)i * NPOS;
            const double* sg_in = A.s.sums + (int64_t)i * NSUM;
            double rp[RP], rs[RS], rk[RK];
#pragma unroll
            for (int r = 0; r < RP; ++r) rp[r] = lane + 32 * r < NPOS ? posg[lane + 32 * r] : 0.0;
#pragma unroll
            for (int r = 0; r < RS; ++r) rs[r] = lane + 32 * r < NSUM ? sg_in[lane + 32 * r] : 0.0;
            const double* Kl = A.c.kinv + (int64_t)level * nk * nk;
#pragma unroll
            for (int r = 0; r < RK; ++r) rk[r] = lane + 32 * r < nk * nk ? ld_const(Kl + lane + 32 * r) : 0.0;
            const double* qg = A.c.q + (int64_t)i * DIM * m;
            const double* bg = A.c.bvals + (int64_t)i * DIM * ne;
            const double q0 = lane < DIM * m ? qg[lane] : 0.0;
            const double q1 = lane + 32 < DIM * m ? qg[lane + 32] : 0.0;
            const double bv0 = lane < DIM * ne ? bg[lane] : 0.0;
            const double bv1 = lane + 32 < DIM * ne ? bg[lane + 32] : 0.0;
            // the member's bookkeeping (the epilogue's stall rule then reads no global memory)
            const int w2 = 2 * A.p.stall_window;
            const double rg0 = lane < w2 ? A.s.ring[(int64_t)i * w2 + lane] : 0.0;
            const double rg1 = lane + 32 < w2 ? A.s.ring[(int64_t)i * w2 + lane + 32] : 0.0;
            if (lane == 0) {
                S->rho = A.s.rho[i];
                S->rho_o = A.s.rho_o[i];
                S->status = A.s.status[i];
                S->level = level;
                S->iteration = A.s.iteration[i];
                S->n_hist = A.s.n_hist[i];
                S->last_change = A.s.last_change[i];
                S->n_changes = A.s.n_changes[i];
            }
#pragma unroll
            for (int r = 0; r < RP; ++r)
                if (lane + 32 * r < NPOS) pPrev[lane + 32 * r] = rp[r];
#pragma unroll
            for (int r = 0; r < RS; ++r)
                if (lane + 32 * r < NSUM) sSumIn[lane + 32 * r] = rs[r];
#pragma unroll
            for (int r = 0; r < RK; ++r)
                if (lane + 32 * r < nk * nk) sK[lane + 32 * r] = rk[r];
            if (lane < DIM * m) sQ[lane] = q0;
            if (lane + 32 < DIM * m) sQ[lane + 32] = q1;
            if (lane < DIM * ne) sBv[lane] = bv0;
            if (lane + 32 < DIM * ne) sBv[lane + 32] = bv1;
            if (lane < w2) S->ring[lane] = rg0;
            if (lane + 32 < w2) S->ring[lane + 32] = rg1;
            __syncwarp();
            const double rho_o = S->rho_o;
            // q_lin[ax][c] = (q + sum_t Slam[ax][t] P[t][c]) - sum_t (rho_o ST[ax][t]) P[t][c]: one lane per output,
            // four interleaved partial sums per product (t = 4k + r), combined (0 + 1) + (2 + 3)
            for (int o = lane; o < DIM * m; o += 32) {
                const int ax = o / m, cc = o - ax * m;
                const double* sl = sSumIn + ax * NP;
                const double* st = sSumIn + (DIM + ax) * NP;
                double u[4] = {0.0, 0.0, 0.0, 0.0}, v[4] = {0.0, 0.0, 0.0, 0.0};
#pragma unroll 5
                for (int tt = 0; tt < NP; tt += 4) {
#pragma unroll
                    for (int r = 0; r < 4; ++r) {
                        if (tt + r < NP) {
                            const double pt = sP[(tt + r) * m + cc];
                            u[r] = fma(sl[tt + r], pt, u[r]);
                            v[r] = fma(rho_o * st[tt + r], pt, v[r]);
                        }
                    }
                }
                sQlin[o] = (sQ[o] + ((u[0] + u[1]) + (u[2] + u[3]))) - ((v[0] + v[1]) + (v[2] + v[3]));
            }
            __syncwarp();
            // xi = K^-1 [-q_lin ; b]  (first m rows of the saddle solution, qpcore.py:141-143)
            for (int o = lane; o < DIM * m; o += 32) {
                const int ax = o / m, r = o - ax * m;
                const double* Kr = sK + r * nk;
                double acc = 0.0;
                for (int cc = 0; cc < m; ++cc) acc += Kr[cc] * (-sQlin[ax * m + cc]);
                for (int e = 0; e < ne; ++e) acc += Kr[m + e] * sBv[ax * ne + e];
                xs[o] = acc;
                if (!split) A.s.xi[(int64_t)i * DIM * m + o] = acc;  // split: written by the combining half
            }
            __syncwarp();
            for (int k = lane; k < NPOS; k += 32) {
                const int ax = k / NP, tt = k - ax * NP;
                double acc = 0.0;
                for (int cc = 0; cc < m; ++cc) acc += sP[tt * m + cc] * xs[ax * m + cc];
                pNew[k] = acc;
                if (!split) A.s.pos[(int64_t)i * NPOS + k] = acc;
            }
            if (lane == 0) {
                sScal[2 * b] = S->rho;
                sScal[2 * b + 1] = rho_o;
            }
            __syncwarp();
            if (lane == 0) mbar_arrive(&ready[b]);
        };
        auto epilogue = [&](const WorkUnit& wu, int b) {
            const int i = wu.member;
            const double* red = sRed + b * kRedBuf;
            const double* wp = sWarp + b * 2 * NCW;
            SchedS* S = reinterpret_cast<SchedS*>(reinterpret_cast<unsigned char*>(sSched) + b * kSchedBytes);
            const int status0 = S->status;
            const int level = S->level;
            const double rho = sScal[2 * b], rho_o = sScal[2 * b + 1];
            if (wu.half < 0) {
                double* sg = A.s.sums + (int64_t)i * 2 * DIM * NP;
                for (int k = lane; k < 2 * DIM * NP; k += 32) {
                    double acc = 0.0;
                    for (int gg = 0; gg < G; ++gg) acc += red[gg * 2 * DIM * NP + k];
                    sg[k] = k < DIM * NP ? acc : acc + sTrk[k - DIM * NP];
                }
                if (lane == 0) {
                    double ss = 0.0, mm = 0.0;
                    for (int w = 0; w < NCW; ++w) {
                        ss += wp[w];
                        mm = fmax(mm, wp[NCW + w]);
                    }
                    if (ss != ss) mm = ss;  // np.max propagates NaN
                    alg1_schedule(A, i, status0, level, rho, rho_o, sqrt(ss), mm, S);
                }
                __syncwarp();
                return;
            }
            // tail half: this half's sums over its groups, residual sum of squares and max into the scratch;
            // the second half to finish combines (half 0 + half 1: a fixed order whichever finishes last)
            constexpr int kPart = 2 * DIM * NP + 2;
            const int tk = wu.pos - rounds * (int)gridDim.x;  // tail index in the work list
            double* part = A.s.split_scratch + ((int64_t)tk * 2 + wu.half) * kPart;
            for (int k = lane; k < 2 * DIM * NP; k += 32) {
                double acc = 0.0;
                for (int gg = 0; gg < G; ++gg) acc += red[gg * 2 * DIM * NP + k];
                part[k] = acc;
            }
            if (lane == 0) {
                double ss = 0.0, mm = 0.0;
                for (int w = 0; w < NCW; ++w) {
                    ss += wp[w];
                    mm = fmax(mm, wp[NCW + w]);
                }
                part[2 * DIM * NP] = ss;
                part[2 * DIM * NP + 1] = mm;
            }
            __threadfence();
            __syncwarp();
            int last = 0;
            if (lane == 0) last = atomicAdd(A.s.split_ticket + tk, 1u) == 1u;
            last = __shfl_sync(0xffffffffu, last, 0);
            if (last) {
                __threadfence();
                const double* p0 = A.s.split_scratch + (int64_t)tk * 2 * kPart;
                const double* p1 = p0 + kPart;
                double* sg = A.s.sums + (int64_t)i * 2 * DIM * NP;
                const double* pNew = sPosNew + b * DIM * NP;
                const double* xs = sXi + b * DIM * 16;
                for (int k = lane; k < 2 * DIM * NP; k += 32) {
                    const double h = __ldcg(p0 + k) + __ldcg(p1 + k);
                    sg[k] = k < DIM * NP ? h : h + sTrk[k - DIM * NP];
                }
                for (int k = lane; k < DIM * NP; k += 32) A.s.pos[(int64_t)i * DIM * NP + k] = pNew[k];
                for (int k = lane; k < DIM * m; k += 32) A.s.xi[(int64_t)i * DIM * m + k] = xs[k];
                if (lane == 0) {
                    const double ss = __ldcg(p0 + 2 * DIM * NP) + __ldcg(p1 + 2 * DIM * NP);
                    double mm = fmax(__ldcg(p0 + 2 * DIM * NP + 1), __ldcg(p1 + 2 * DIM * NP + 1));
                    if (ss != ss) mm = ss;  // np.max propagates NaN
                    alg1_schedule(A, i, status0, level, rho, rho_o, sqrt(ss), mm, S);
                    A.s.split_ticket[tk] = 0u;  // ready for the next launch
                }
            }
            __syncwarp();
        };

        WorkUnit pw, ew;
        int pu = next_active(A, 0, n_units, rounds, split_tail, nst, order, &pw);
        for (int pk = 0; pk < 2 && pu < n_units; ++pk) {  // prime both buffers
            prologue(pw, pk);
            pu = next_active(A, pu + 1, n_units, rounds, split_tail, nst, order, &pw);
        }
        int ek = 0;
        for (int eu = next_active(A, 0, n_units, rounds, split_tail, nst, order, &ew); eu < n_units;
             eu = next_active(A, eu + 1, n_units, rounds, split_tail, nst, order, &ew), ++ek) {
            const int b = ek & 1;
            mbar_wait(&done[b], (uint32_t)((ek >> 1) & 1));
            epilogue(ew, b);
            if (pu < n_units) {  // buffer b is free again: the prologue two units ahead
                prologue(pw, b);
                pu = next_active(A, pu + 1, n_units, rounds, split_tail, nst, order, &pw);
            }
        }
        return;
    }

    // ======================= consumers
    const int t = tid % NP;
    const int g = tid / NP;
    const bool act = g < G;
    int s = 0;
    uint32_t ph = 0;
    // this thread's offsets inside a stage: its obstacle row of state and of tracks, sample t
    const int row_off = g * C::kRowBytes + t * (int)sizeof(T);
    const int trk_off = G * C::kRowBytes + g * C::kTrkBytes + t * 8;
    const double rel_t = lin ? sLin[6 * n_o + t] : 0.0;  // this sample's time offset (linear tracks)
    const int64_t Nel = (int64_t)B * n_o * NP;
    T* dst = EXP ? reinterpret_cast<T*>(A.s.d) : nullptr;
    T* cop = EXP ? reinterpret_cast<T*>(A.s.copies) : nullptr;

    WorkUnit wu;
    int k = 0;
    for (int u = next_active(A, 0, n_units, rounds, split_tail, nst, order, &wu); u < n_units;
         u = next_active(A, u + 1, n_units, rounds, split_tail, nst, order, &wu), ++k) {
        const int i = wu.member;
        const int b = k & 1;
        mbar_wait(&ready[b], (uint32_t)((k >> 1) & 1));  // the scalar warp's prologue of this unit
        const double rho = sScal[2 * b], rho_o = sScal[2 * b + 1];
        const double* pNew = sPosNew + b * DIM * NP;
        const double* pPrev = sPosPrev + b * DIM * NP;

        // ---------- element pass out of the shared-memory ring
        // per-thread accumulation in the storage type (fp32 builds: no double conversions per element; the
        // partials are widened once per member)
        T sumsq = (T)0, mx = (T)0, accL[DIM], accO[DIM];
#pragma unroll
        for (int ax = 0; ax < DIM; ++ax) accL[ax] = accO[ax] = (T)0;
        const T px = (T)pNew[t], py = (T)pNew[NP + t], pz = DIM == 3 ? (T)pNew[2 * NP + t] : (T)0;
        const T ox = (T)pPrev[t], oy = (T)pPrev[NP + t], oz = DIM == 3 ? (T)pPrev[2 * NP + t] : (T)0;
        const T trho = (T)rho, trho_o = (T)rho_o;
        const int d_mode = DM >= 0 ? DM : A.p.d_mode;
        T* gbase = reinterpret_cast<T*>(A.s.state) + (int64_t)i * n_o * W * NP + t;

        const int j_first = wu.st0 * G + g, j_end = wu.st1 * G + g;  // this unit's stages
        T* gp = gbase + (int64_t)j_first * W * NP;
        int64_t e = ((int64_t)i * n_o + j_first) * NP + t;  // index into the optional d / copies planes
        for (int j = j_first; j < j_end && j - g < n_o; j += G, gp += G * W * NP, e += G * NP) {
            mbar_wait(&full[s], ph);
            if (act && j < n_o) {
                const unsigned char* buf = stages + s * L.stage_bytes;
                const T* row = reinterpret_cast<const T*>(buf + row_off);
                T v[W];
#pragma unroll
                for (int w = 0; w < W; ++w) v[w] = row[w * NP];
                T trx, trY, trz;
                if (lin) {
                    if constexpr (sizeof(T) == 8) {  // c + v rel_t rounded like numpy's c + v * rel (bitwise)
                        const double* lj = sLin + 6 * j;  // 3-D {cx cy cz vx vy vz}, 2-D {cx cy vx vy - -}
                        const double2 q0 = *reinterpret_cast<const double2*>(lj);
                        const double2 q1 = *reinterpret_cast<const double2*>(lj + 2);
                        if constexpr (DIM == 3) {
                            const double2 q2 = *reinterpret_cast<const double2*>(lj + 4);
                            trx = __dadd_rn(q0.x, __dmul_rn(q1.y, rel_t));
                            trY = __dadd_rn(q0.y, __dmul_rn(q2.x, rel_t));
                            trz = __dadd_rn(q1.x, __dmul_rn(q2.y, rel_t));
                        } else {
                            trx = __dadd_rn(q0.x, __dmul_rn(q1.x, rel_t));
                            trY = __dadd_rn(q0.y, __dmul_rn(q1.y, rel_t));
                            trz = 0.0;
                        }
                    } else {  // fp32 build: the track in float (1e-4 contract)
                        const float* lj = sLinF + 6 * j;
                        const float relf = (float)rel_t;
                        const float2 q0 = *reinterpret_cast<const float2*>(lj);
                        const float2 q1 = *reinterpret_cast<const float2*>(lj + 2);
                        const float2 q2 = *reinterpret_cast<const float2*>(lj + 4);
                        if constexpr (DIM == 3) {
                            trx = fmaf(q1.y, relf, q0.x);
                            trY = fmaf(q2.x, relf, q0.y);
                            trz = fmaf(q2.y, relf, q1.x);
                        } else {
                            trx = fmaf(q1.x, relf, q0.x);
                            trY = fmaf(q1.y, relf, q0.y);
                            trz = 0.0f;
                        }
                    }
                } else {
                    const double* trow = reinterpret_cast<const double*>(buf + trk_off);
                    trx = (T)trow[0];
                    trY = (T)trow[NP];
                    trz = DIM == 3 ? (T)trow[2 * NP] : (T)0;
                }
                T a, bb, ia2, ib2;
                if constexpr (sizeof(T) == 8) {
                    const double2 ab = *reinterpret_cast<const double2*>(sShp + 4 * j);
                    const double2 iab = *reinterpret_cast<const double2*>(sShp + 4 * j + 2);
                    a = ab.x; bb = ab.y; ia2 = iab.x; ib2 = iab.y;
                } else {
                    const float4 sh = *reinterpret_cast<const float4*>(sShpF + 4 * j);
                    a = sh.x; bb = sh.y; ia2 = sh.z; ib2 = sh.w;
                }
                T dold;
                if (d_mode == 0) {
                    dold = (T)1;
                } else if (EXP && d_mode == 1) {
                    dold = dst[e];
                } else {
                    const T ex = ox - trx, ey = oy - trY;
                    T qd;
                    if constexpr (DIM == 3) {
                        const T ez = oz - trz;
                        qd = ex * ex * ia2 + ey * ey * ia2 + ez * ez * ib2;
                    } else {
                        qd = ex * ex * ia2 + ey * ey * ib2;
                    }
                    dold = los_scale(qd);
                }
                T dn, cp4[4], ss, ml, off[DIM];
                am_element<DIM, T, LAY>(v, px - trx, py - trY, pz - trz, a, bb, ia2, ib2, dold, trho, trho_o, ss, ml,
                                        off, dn, cp4);
                sumsq += ss;
                mx = ml > mx ? ml : mx;
#pragma unroll
                for (int ax = 0; ax < DIM; ++ax) {
                    accL[ax] += v[Words<DIM, LAY>::NV + ax];
                    accO[ax] += off[ax];
                }
#pragma unroll
                for (int w = 0; w < W; ++w) st_stream(gp + w * NP, v[w]);
                if constexpr (EXP) {
                    if (dst) dst[e] = dn;  // optional exports (tests, warm starts)
                    if (cop) {
#pragma unroll
                        for (int c = 0; c < 2 * (DIM - 1); ++c) cop[c * Nel + e] = cp4[c];
                    }
                }
            }
            __syncwarp();
            if (lane == 0) mbar_arrive(&empty[s]);
            if (++s == S) {
                s = 0;
                ph ^= 1u;
            }
        }

        // ---------- hand the partials to the scalar warp (fixed-order reductions there)
        double* red = sRed + b * kRedBuf;
        if (act) {
#pragma unroll
            for (int ax = 0; ax < DIM; ++ax) {
                red[(g * 2 * DIM + ax) * NP + t] = (double)accL[ax];
                red[(g * 2 * DIM + DIM + ax) * NP + t] = (double)accO[ax];
            }
        }
        const double wss = warp_sum((double)sumsq);
        const double wmx = warp_max((double)mx);
        if (lane == 0) {
            sWarp[b * 2 * NCW + warp] = wss;
            sWarp[b * 2 * NCW + NCW + warp] = wmx;
        }
        __syncwarp();
        if (lane == 0) mbar_arrive(&done[b]);
    }
}

}  // namespace tro
