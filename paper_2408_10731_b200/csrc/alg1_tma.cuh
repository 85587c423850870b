// Persistent, warp-specialised fused AM iteration (Alg. 1) for sm_100a.
//
// Why: the one-CTA-per-member kernel is latency-bound — each warp issues its
// element's 12 global loads and then computes ~500 instructions with nothing in
// flight, so too few bytes are outstanding per SM (ncu: long-scoreboard stalls
// dominate, 0.6 eligible warps/cycle).  Here one producer warp streams the
// state rows into a shared-memory ring with TMA bulk copies
// (cp.async.bulk ... mbarrier::complete_tx) while G*NP consumer threads compute
// out of shared memory and write results straight back to HBM.  In the
// interleaved layout state[i][j][w][t] the W words x NP samples of one
// obstacle row are ONE contiguous block (fp64 3-D: 7200 B), as is the matching
// track row tracks[j][ax][t], so a stage (G rows) is 2G bulk copies.
//
// Grid = min(B, SMs): each CTA walks members i = blockIdx.x, += gridDim.x and
// the producer runs ahead across member boundaries, so the next member's first
// rows are in flight while the consumers do this member's epilogue and the
// next member's QP prologue.  Consumers synchronise with a named barrier
// (bar 1) that excludes the producer warp.
#pragma once
#include "alg1_elem.cuh"
#include "tma.cuh"

namespace tro {

template <int DIM, typename T, int LAY, int NP, int G, int S>
struct TmaCfg {
    static constexpr int W = Words<DIM, LAY>::W;
    static constexpr int kRowBytes = W * NP * (int)sizeof(T);  // one obstacle row of state
    static constexpr int kTrkBytes = DIM * NP * 8;             // one obstacle row of tracks
    static constexpr int kStageBytes = G * (kRowBytes + kTrkBytes);
    static constexpr int kConsumers = ((G * NP + 31) / 32) * 32;
    static constexpr int kThreads = kConsumers + 32;
    static_assert(kRowBytes % 16 == 0 && kTrkBytes % 16 == 0, "bulk copies need 16-byte rows");
};

// shared-memory carve-up (bytes): [stages | P | pos_prev | pos_new | sums_in | red | shapes | qlin | xi | warp | bars]
struct TmaLayout {
    int stages, P, pos_prev, pos_new, sums_in, red, shp, qlin, xi, warp, bars, total;
};
__host__ __device__ inline TmaLayout tma_layout(int stage_bytes, int S, int n_p, int m, int dim, int n_o, int G,
                                                int consumers) {
    TmaLayout L;
    int off = 0;
    L.stages = off; off += S * stage_bytes;
    L.P = off;        off += n_p * m * 8;
    L.pos_prev = off; off += dim * n_p * 8;
    L.pos_new = off;  off += dim * n_p * 8;
    L.sums_in = off;  off += 2 * dim * n_p * 8;
    L.red = off;      off += G * 2 * dim * n_p * 8;
    off = (off + 15) & ~15;
    L.shp = off;      off += 4 * (n_o > 0 ? n_o : 1) * 8;  // per obstacle {a, b, 1/a^2, 1/b^2} (two 16-B loads)
    L.qlin = off;     off += dim * 16 * 8;
    L.xi = off;       off += dim * 16 * 8;
    L.warp = off;     off += 2 * (consumers / 32) * 8;
    off = (off + 15) & ~15;
    L.bars = off;     off += 2 * S * 8;
    L.total = off;
    return L;
}

#ifndef TRO_TMA_MINB
#define TRO_TMA_MINB 2
#endif
constexpr int kTmaMinBlocks = TRO_TMA_MINB;  // resident CTAs per SM the kernel is compiled for

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

// DM: the previous iterate's d source fixed at compile time (2: recompute, the steady state) or -1 (read
// A.p.d_mode at run time: the first iteration after an init / prime)
template <int DIM, typename T, int LAY, int NP, int G, int S, int DM>
__global__ void __launch_bounds__(TmaCfg<DIM, T, LAY, NP, G, S>::kThreads, kTmaMinBlocks) alg1_tma_kernel(Alg1Args A) {
    using C = TmaCfg<DIM, T, LAY, NP, G, S>;
    constexpr int W = C::W;
    constexpr int NC = C::kConsumers;
    constexpr int NCW = NC / 32;
    extern __shared__ __align__(128) unsigned char smraw[];
    const int n_o = A.d.n_obs, m = A.d.m, ne = A.d.n_eq, nk = m + ne;
    const int B = A.d.n_members;
    const TmaLayout L = tma_layout(C::kStageBytes, S, NP, m, DIM, n_o, G, NC);
    unsigned char* stages = smraw + L.stages;
    double* sP = reinterpret_cast<double*>(smraw + L.P);
    double* sPosPrev = reinterpret_cast<double*>(smraw + L.pos_prev);
    double* sPosNew = reinterpret_cast<double*>(smraw + L.pos_new);
    double* sSumIn = reinterpret_cast<double*>(smraw + L.sums_in);
    double* sRed = reinterpret_cast<double*>(smraw + L.red);
    double* sShp = reinterpret_cast<double*>(smraw + L.shp);
    double* sQlin = reinterpret_cast<double*>(smraw + L.qlin);
    double* sXi = reinterpret_cast<double*>(smraw + L.xi);
    double* sWarp = reinterpret_cast<double*>(smraw + L.warp);
    uint64_t* full = reinterpret_cast<uint64_t*>(smraw + L.bars);
    uint64_t* empty = full + S;

    const int tid = threadIdx.x;
    const int warp = tid >> 5, lane = tid & 31;

    // ---------------- one-time setup: barriers, basis, shapes
    if (tid == 0) {
        for (int s = 0; s < S; ++s) {
            mbar_init(&full[s], 1);
            mbar_init(&empty[s], NCW);
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
    __syncthreads();

    const int nst = (n_o + G - 1) / G;  // stages per member
    // ring position: stage s and its phase bit run on across members (no divisions in the loops)
    // work units of this CTA: members blockIdx.x + u gridDim.x, or with tail balancing (A.split_tail = M > 0)
    // `rounds` full rounds and then, for the first 2 M CTAs, one half (of the stages) of a tail member
    // the work list: order[0 .. *n_order) when given (e.g. the robots still driving), else members 0..B-1
    const int32_t* order = A.s.order;
    const int n_work = order ? *A.s.n_order : B;
    const int rounds = n_work / (int)gridDim.x;
    const int tail = n_work - rounds * (int)gridDim.x;
    const int split_tail = (A.split_tail && tail > 0 && 2 * tail <= (int)gridDim.x) ? tail : 0;
    const int n_units = split_tail ? rounds + ((int)blockIdx.x < 2 * split_tail ? 1 : 0)
                                   : (n_work - (int)blockIdx.x + (int)gridDim.x - 1) / (int)gridDim.x;

    if (warp == NCW) {
        // ======================= producer warp (one elected lane)
        if (lane == 0) {
            int s = 0;
            uint32_t ph = 0;
            bool wrapped = false;
            for (int u = 0; u < n_units; ++u) {
                const WorkUnit wu = work_unit(u, rounds, split_tail, nst, order);
                const int i = wu.member;
                const int st = A.s.status[i];
                if ((st & (TRO_CONVERGED | TRO_FACTOR_FAILED)) || !A.c.level_ok[A.s.level[i]]) continue;
                const unsigned char* src = reinterpret_cast<const unsigned char*>(A.s.state) +
                                           (int64_t)i * n_o * C::kRowBytes;
                const unsigned char* trk = reinterpret_cast<const unsigned char*>(A.c.tracks);
                for (int j0 = wu.st0 * G; j0 < n_o && j0 < wu.st1 * G; j0 += G) {
                    if (wrapped) mbar_wait(&empty[s], ph ^ 1u);  // the consumers released this stage
                    const int rows = min(G, n_o - j0);
                    unsigned char* buf = stages + s * C::kStageBytes;
                    mbar_expect_tx(&full[s], rows * (C::kRowBytes + C::kTrkBytes));
                    bulk_g2s(buf, src + (int64_t)j0 * C::kRowBytes, rows * C::kRowBytes, &full[s]);
                    bulk_g2s(buf + G * C::kRowBytes, trk + (int64_t)j0 * C::kTrkBytes, rows * C::kTrkBytes, &full[s]);
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

    // ======================= consumers
    const int t = tid % NP;
    const int g = tid / NP;
    const bool act = g < G;
    int s = 0;
    uint32_t ph = 0;
    // this thread's offsets inside a stage: its obstacle row of state and of tracks, sample t
    const int row_off = g * C::kRowBytes + t * (int)sizeof(T);
    const int trk_off = G * C::kRowBytes + g * C::kTrkBytes + t * 8;
    const int64_t Nel = (int64_t)B * n_o * NP;
    T* dst = reinterpret_cast<T*>(A.s.d);
    T* cop = reinterpret_cast<T*>(A.s.copies);

    for (int u = 0; u < n_units; ++u) {
        const WorkUnit wu = work_unit(u, rounds, split_tail, nst, order);
        const int i = wu.member;
        const bool split = wu.half >= 0;
        const int status0 = A.s.status[i];
        if (status0 & (TRO_CONVERGED | TRO_FACTOR_FAILED)) continue;
        const int level = A.s.level[i];
        if (!A.c.level_ok[level]) {  // qpcore.py:108-110 -> the host raises FactorizationError
            if (tid == 0) A.s.status[i] = status0 | TRO_FACTOR_FAILED;
            continue;
        }
        const double rho = A.s.rho[i];
        const double rho_o = A.s.rho_o[i];

        // ---------- QP position step (solver_single.py:204-211)
        const double* posg = A.s.pos + (int64_t)i * DIM * NP;
        for (int k = tid; k < DIM * NP; k += NC) sPosPrev[k] = posg[k];
        const double* sg_in = A.s.sums + (int64_t)i * 2 * DIM * NP;
        for (int k = tid; k < 2 * DIM * NP; k += NC) sSumIn[k] = sg_in[k];
        consumer_sync(NC);
        const double* qg = A.c.q + (int64_t)i * DIM * m;
        for (int o = warp; o < DIM * m; o += NCW) {
            const int ax = o / m, cc = o - ax * m;
            double u = 0.0, v = 0.0;
            for (int tt = lane; tt < NP; tt += 32) {
                const double pt = sP[tt * m + cc];
                u += sSumIn[ax * NP + tt] * pt;
                v += (rho_o * sSumIn[(DIM + ax) * NP + tt]) * pt;
            }
            u = warp_sum(u);
            v = warp_sum(v);
            if (lane == 0) sQlin[o] = (qg[o] + u) - v;
        }
        consumer_sync(NC);
        const double* Kl = A.c.kinv + (int64_t)level * nk * nk;
        const double* bg = A.c.bvals + (int64_t)i * DIM * ne;
        for (int o = tid; o < DIM * m; o += NC) {
            const int ax = o / m, r = o - ax * m;
            const double* Kr = Kl + r * nk;
            double acc = 0.0;
            for (int cc = 0; cc < m; ++cc) acc += ld_const(Kr + cc) * (-sQlin[ax * m + cc]);
            for (int e = 0; e < ne; ++e) acc += ld_const(Kr + m + e) * bg[ax * ne + e];
            sXi[o] = acc;
            if (!split) A.s.xi[(int64_t)i * DIM * m + o] = acc;  // split: written by the combining half
        }
        consumer_sync(NC);
        for (int k = tid; k < DIM * NP; k += NC) {
            const int ax = k / NP, tt = k - ax * NP;
            double acc = 0.0;
            for (int cc = 0; cc < m; ++cc) acc += sP[tt * m + cc] * sXi[ax * m + cc];
            sPosNew[k] = acc;
            if (!split) A.s.pos[(int64_t)i * DIM * NP + k] = acc;
        }
        consumer_sync(NC);

        // ---------- element pass out of the shared-memory ring
        double sumsq = 0.0, mx = 0.0;
        double accL[DIM], accT[DIM];
#pragma unroll
        for (int ax = 0; ax < DIM; ++ax) accL[ax] = accT[ax] = 0.0;
        const double px = sPosNew[t], py = sPosNew[NP + t], pz = DIM == 3 ? sPosNew[2 * NP + t] : 0.0;
        const double ox = sPosPrev[t], oy = sPosPrev[NP + t], oz = DIM == 3 ? sPosPrev[2 * NP + t] : 0.0;
        const T trho = (T)rho, trho_o = (T)rho_o;
        const int d_mode = DM >= 0 ? DM : A.p.d_mode;
        T* gbase = reinterpret_cast<T*>(A.s.state) + (int64_t)i * n_o * W * NP + t;

        const int j_first = wu.st0 * G + g, j_end = wu.st1 * G + g;  // this unit's stages
        T* gp = gbase + (int64_t)j_first * W * NP;
        int64_t e = ((int64_t)i * n_o + j_first) * NP + t;  // index into the optional d / copies planes
        for (int j = j_first; j < j_end && j - g < n_o; j += G, gp += G * W * NP, e += G * NP) {
            mbar_wait(&full[s], ph);
            if (act && j < n_o) {
                const unsigned char* buf = stages + s * C::kStageBytes;
                const T* row = reinterpret_cast<const T*>(buf + row_off);
                const double* trow = reinterpret_cast<const double*>(buf + trk_off);
                T v[W];
#pragma unroll
                for (int w = 0; w < W; ++w) v[w] = row[w * NP];
                const double trx = trow[0], trY = trow[NP], trz = DIM == 3 ? trow[2 * NP] : 0.0;
                const double2 ab = *reinterpret_cast<const double2*>(sShp + 4 * j);
                const double2 iab = *reinterpret_cast<const double2*>(sShp + 4 * j + 2);
                const T a = (T)ab.x, b = (T)ab.y, ia2 = (T)iab.x, ib2 = (T)iab.y;
                T dold;
                if (d_mode == 0) {
                    dold = (T)1;
                } else if (d_mode == 1) {
                    dold = dst[e];
                } else {
                    const T ex = (T)(ox - trx), ey = (T)(oy - trY);
                    T qd;
                    if constexpr (DIM == 3) {
                        const T ez = (T)(oz - trz);
                        qd = ex * ex * ia2 + ey * ey * ia2 + ez * ez * ib2;
                    } else {
                        qd = ex * ex * ia2 + ey * ey * ib2;
                    }
                    dold = los_scale(qd);
                }
                T dn, cp4[4];
                am_element<DIM, T, LAY>(v, trx, trY, trz, px, py, pz, a, b, ia2, ib2, dold, trho, trho_o, sumsq, mx,
                                   accL, accT, dn, cp4);
#pragma unroll
                for (int w = 0; w < W; ++w) st_stream(gp + w * NP, v[w]);
                if (dst) dst[e] = dn;  // optional exports (tests, warm starts)
                if (cop) {
#pragma unroll
                    for (int c = 0; c < 2 * (DIM - 1); ++c) cop[c * Nel + e] = cp4[c];
                }
            }
            __syncwarp();
            if (lane == 0) mbar_arrive(&empty[s]);
            if (++s == S) {
                s = 0;
                ph ^= 1u;
            }
        }

        // ---------- epilogue (fixed-order reductions, history, stall rule)
        if (act) {
#pragma unroll
            for (int ax = 0; ax < DIM; ++ax) {
                sRed[(g * 2 * DIM + ax) * NP + t] = accL[ax];
                sRed[(g * 2 * DIM + DIM + ax) * NP + t] = accT[ax];
            }
        }
        sumsq = warp_sum(sumsq);
        mx = warp_max(mx);
        if (lane == 0) {
            sWarp[warp] = sumsq;
            sWarp[NCW + warp] = mx;
        }
        consumer_sync(NC);
        if (!split) {
            double* sg = A.s.sums + (int64_t)i * 2 * DIM * NP;
            for (int k = tid; k < 2 * DIM * NP; k += NC) {
                double acc = 0.0;
                for (int gg = 0; gg < G; ++gg) acc += sRed[gg * 2 * DIM * NP + k];
                sg[k] = acc;
            }
            if (tid == 0) {
                double ss = 0.0, mm = 0.0;
                for (int w = 0; w < NCW; ++w) {
                    ss += sWarp[w];
                    mm = fmax(mm, sWarp[NCW + w]);
                }
                if (ss != ss) mm = ss;  // np.max propagates NaN
                alg1_schedule(A, i, status0, level, rho, rho_o, sqrt(ss), mm);
            }
        } else {
            // this half's sums over its groups, residual sum of squares and max into the scratch; the
            // second half to finish combines (half 0 + half 1: a fixed order whichever finishes last)
            constexpr int kPart = 2 * DIM * NP + 2;
            const int tk = wu.pos - rounds * (int)gridDim.x;  // tail index in the work list
            double* part = A.s.split_scratch + ((int64_t)tk * 2 + wu.half) * kPart;
            for (int k = tid; k < 2 * DIM * NP; k += NC) {
                double acc = 0.0;
                for (int gg = 0; gg < G; ++gg) acc += sRed[gg * 2 * DIM * NP + k];
                part[k] = acc;
            }
            __shared__ int sLast;
            if (tid == 0) {
                double ss = 0.0, mm = 0.0;
                for (int w = 0; w < NCW; ++w) {
                    ss += sWarp[w];
                    mm = fmax(mm, sWarp[NCW + w]);
                }
                part[2 * DIM * NP] = ss;
                part[2 * DIM * NP + 1] = mm;
            }
            consumer_sync(NC);
            if (tid == 0) {
                __threadfence();
                sLast = atomicAdd(A.s.split_ticket + tk, 1u) == 1u;
            }
            consumer_sync(NC);
            if (sLast) {
                __threadfence();
                const double* p0 = A.s.split_scratch + (int64_t)tk * 2 * kPart;
                const double* p1 = p0 + kPart;
                double* sg = A.s.sums + (int64_t)i * 2 * DIM * NP;
                for (int k = tid; k < 2 * DIM * NP; k += NC) sg[k] = __ldcg(p0 + k) + __ldcg(p1 + k);
                for (int k = tid; k < DIM * NP; k += NC) A.s.pos[(int64_t)i * DIM * NP + k] = sPosNew[k];
                for (int k = tid; k < DIM * m; k += NC) A.s.xi[(int64_t)i * DIM * m + k] = sXi[k];
                if (tid == 0) {
                    const double ss = __ldcg(p0 + 2 * DIM * NP) + __ldcg(p1 + 2 * DIM * NP);
                    double mm = fmax(__ldcg(p0 + 2 * DIM * NP + 1), __ldcg(p1 + 2 * DIM * NP + 1));
                    if (ss != ss) mm = ss;  // np.max propagates NaN
                    alg1_schedule(A, i, status0, level, rho, rho_o, sqrt(ss), mm);
                    A.s.split_ticket[tk] = 0u;  // ready for the next launch
                }
            }
        }
        consumer_sync(NC);  // sRed / sWarp / sPos* are reused by the next member
    }
}

}  // namespace tro
