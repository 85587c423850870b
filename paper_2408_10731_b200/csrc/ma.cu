// Batched joint multi-agent AM iteration (arXiv 2408.10731, Alg. 5) for sm_100a.
//
// One CTA owns one joint problem (N_a agents, n_pairs = N_a(N_a-1)/2 agent pairs +
// N_a per static sphere) for one iteration of solve_joint (solver_multiagent.py:252-335):
//   prologue : the per-axis QP, xi = K_L^-1 [ rho A'B - A'C ; b_eq ], from the agent-
//              contracted sums B (recon + statics) and C (lambda) the previous launch left
//              behind (b_fo = recon - lambda/rho + statics, :266-268) -- or, mode 4, the xi the
//              batched tensor-core QP kernel (ma_qp_kernel) wrote; the boundary projection;
//   body     : rounds of kMaWarps samples, warp w on t = r kMaWarps + w: the sample's positions,
//              then lanes over pairs (state[i][t][w][p], pairs fastest: coalesced).  Per (pair, t):
//              alpha/beta of the new offsets in trig-free form (unit vectors), the multiplier-shifted
//              d (:285-293), residual and multiplier ascent (:295-296).  Only the multipliers persist:
//              alpha, beta come from the positions and d only feeds the next RHS, folded into the sums;
//              each pair's recon and lambda are scattered to its two agents through colour-ordered
//              incidence lists (fixed order) into the round's V rows;
//   contract : V (agent sums x samples) times P on the fp64 tensor cores (DMMA tiles owned by warps,
//              accumulated across rounds; rounds handed over through mbarriers);
//   epilogue : the sums B, C for the next launch; residual norm / max; history; the staged level
//              schedule (:313-335).
// Deterministic: every reduction has a fixed order, so a problem's bits do not depend on
// the batch or the GPU count.
#include <type_traits>

#include "common.cuh"
#include "fastmath.cuh"
#include "tma.cuh"
#include "../../include/trajopt_b200.h"

namespace tro {

#ifndef MA_MINB
#define MA_MINB 2  // resident CTAs per SM the element kernel is compiled for (128 registers)
#endif
#ifndef MA_QP_PRE
#define MA_QP_PRE 4  // k-steps of K^-1 fragments in flight in the DMMA QP kernel (2 / 3 / 4 / 6 / 8: 83 / 83 / 69 / 99 / 105 us)
#endif
#ifndef MA_PAIR_UNROLL
#define MA_PAIR_UNROLL 1  // pair chunks per loop trip of the element pass (C3: 1 -> 0.945, 2 -> 1.05, 4 -> 1.40 ms)
#endif
constexpr int kMaPairUnroll = MA_PAIR_UNROLL;
#ifndef MA_WARPS
#define MA_WARPS 10
#endif
constexpr int kMaWarps = MA_WARPS;  // 100 samples = 10 rounds of 10 (C3); 2 CTAs x 10 warps per SM
constexpr int kMaMaxAgents = 32;
constexpr int kMaMaxRing = 64;

// one bulk L2 prefetch of [p, p + bytes) (16-B aligned, bytes a multiple of 16): the lambda rows of the
// rounds ahead, so the per-lane one-element-ahead loads hit L2 instead of waiting on HBM
__device__ __forceinline__ void prefetch_l2(const void* p, uint32_t bytes) {
    asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(p), "r"(bytes) : "memory");
}
#ifndef MA_AHEAD
#define MA_AHEAD 2
#endif
constexpr int kMaAhead = MA_AHEAD;  // rounds of lambda rows prefetched into L2 ahead of the element pass

// D(8x8) += A(8x4, row) B(4x8, col) in fp64 on the tensor cores (lane l: A[l/4][l%4], B[l%4][l/4],
// D[l/4][2 (l%4) + {0, 1}])
__device__ __forceinline__ void dmma884(double* d, double a, double b) {
    asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0, %1}, {%2}, {%3}, {%0, %1};"
                 : "+d"(d[0]), "+d"(d[1])
                 : "d"(a), "d"(b));
}

struct MaArgs {
    tro_ma_dims d;
    tro_ma_consts c;
    tro_ma_state s;
    tro_ma_params p;
};

struct MaSmem {
    int P, xi, pos, scratch, sumin, rhs, V, warp, pair, ints, total;  // doubles
};
constexpr int kPairW = 7;  // per pair: a, b, 1/a, 1/b, static centre (3)
// scatter scratch, one record per pair: recon + static (x y z), lambda (x y z), one pad double.  The odd
// 56-byte stride keeps the element pass's per-lane record writes conflict-free, and the scatter reads a
// record's three components at immediate offsets from one address.
constexpr int kScrW = 7;
// V row stride: 6 n_a agent sums padded to 4 (mod 16) doubles, so the 4 samples (k) of a DMMA A fragment land
// 8 banks apart (rows of 96 put all four on one bank: 4-way conflicts)
__host__ __device__ inline int ma_vstride(int n_a) { return 6 * n_a + ((4 - (6 * n_a) % 16) + 16) % 16; }
__host__ __device__ inline MaSmem ma_layout(int n_p, int m, int n_a, int n_pairs, int n_eq, int n_inc) {
    MaSmem L;
    int off = 0;
    L.P = off;       off += n_p * ((m + 1) & ~1);        // basis rows padded to an even stride (16-B rows)
    L.xi = off;      off += 3 * n_a * m;                 // this launch's coefficients [axis][agent][c]
    L.pos = off;     off += kMaWarps * n_a * 3;          // per warp: its sample's positions [agent][axis]
    L.scratch = off; off += kMaWarps * n_pairs * kScrW;  // per warp: (recon+static, lambda) per pair
    // the fused prologue's buffers (sums in, RHS) are dead before the element pass: they alias the scratch
    const int pro = 2 * n_a * 3 * m + 3 * (n_a * m + n_eq);
    if (pro > kMaWarps * n_pairs * kScrW) off += pro - kMaWarps * n_pairs * kScrW;
    L.sumin = L.scratch;
    L.rhs = L.sumin + 2 * n_a * 3 * m;
    L.V = off;       off += 2 * kMaWarps * ma_vstride(n_a);  // per round, per warp: the scattered agent sums (x2 buffers)
    L.warp = off;    off += 2 * kMaWarps;
    L.pair = off;    off += kPairW * n_pairs;            // SoA [field][pair]
    L.ints = off;    off += (2 * n_pairs + n_a + 1 + n_inc + 1) / 2 + 1;  // pair_i, pair_j, inc_ptr, inc_pair
    L.total = off;
    return L;
}

template <int M, int MODE>
__global__ void __launch_bounds__(kMaWarps * 32, MA_MINB) ma_kernel(MaArgs A) {
    // MODE 0: iteration; 1: prime (sums of a given state: lambda in `state`, d / alpha / beta in
    // the export planes); 2: cold init (straight lines, angles, d = 1, lambda = 0) + sums;
    // 4: iteration whose QP step already ran (ma_qp_kernel wrote xi): the element pass alone
    constexpr int mode = MODE == 4 ? 0 : MODE;
    constexpr bool init = MODE == 2;
    constexpr bool prime = MODE == 1;
    constexpr bool pre_qp = MODE == 4;
    extern __shared__ double smem[];
    const int i = blockIdx.x;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int n_p = A.d.n_p, n_a = A.d.n_agents, np_ = A.d.n_pairs, neq = A.d.n_eq;
    const int m = M ? M : A.d.m;
    const int nv = n_a * m, nk = nv + neq;
    const int n_inc = A.c.inc_ptr[n_a];  // <= 2 n_pairs (the layout's bound)
    const MaSmem L = ma_layout(n_p, m, n_a, np_, neq, 2 * np_);
    double* sP = smem + L.P;
    double* sPair = smem + L.pair;
    int* sPairI = reinterpret_cast<int*>(smem + L.ints);
    int* sPairJ = sPairI + np_;
    int* sIncPtr = sPairJ + np_;
    int* sInc = sIncPtr + n_a + 1;
    double* sPos = smem + L.pos + warp * n_a * 3;
    double* sScr = smem + L.scratch + warp * np_ * kScrW;
    double* sV = smem + L.V;
    double* sSumIn = smem + L.sumin;
    double* sRhs = smem + L.rhs;
    double* sXi = smem + L.xi;
    double* sWarp = smem + L.warp;

    bool uni;  // every pair shares (a, b) and has an agent partner
    const int status0 = A.s.status[i];
    if (mode == 0 && (status0 & TRO_CONVERGED)) return;
    __shared__ uint64_t sBar[4];  // V[0 / 1] published by every warp (full), read by every warp (empty)
    if (tid == 0) {
        for (int k = 0; k < 4; ++k) mbar_init(&sBar[k], kMaWarps);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    if (mode == 0 && lane == 0 && ((3 * np_ * 8) & 15) == 0)  // this warp's first kMaAhead rounds of lambda rows
        for (int r = 0; r < kMaAhead; ++r) {
            const int t = r * kMaWarps + warp;
            if (t < n_p) prefetch_l2(A.s.state + ((int64_t)i * n_p + t) * 3 * np_, 3 * np_ * 8);
        }
    const int level = A.s.level[i];
    const double rho = A.c.level_rho[level];
    const int mp = (m + 1) & ~1;
    for (int k = tid; k < n_p * mp; k += blockDim.x) {
        const int t = k / mp, c = k - t * mp;
        sP[k] = c < m ? ld_const(A.c.P + t * m + c) : 0.0;
    }
    {
        // per-pair constants (no divisions in the element pass) and the incidence lists
        const double* statics_i = A.c.statics ? A.c.statics + (int64_t)i * A.d.n_static * 3 : nullptr;
        for (int p = tid; p < np_; p += blockDim.x) {
            const double pa = A.c.pair_a[p], pb = A.c.pair_b[p];
            const int pj = A.c.pair_j[p];
            sPair[0 * np_ + p] = pa;
            sPair[1 * np_ + p] = pb;
            sPair[2 * np_ + p] = 1.0 / pa;
            sPair[3 * np_ + p] = 1.0 / pb;
            for (int k = 0; k < 3; ++k)
                sPair[(4 + k) * np_ + p] = pj < 0 ? statics_i[A.c.pair_s[p] * 3 + k] : 0.0;
            sPairI[p] = A.c.pair_i[p];
            sPairJ[p] = pj;
        }
        for (int k = tid; k <= n_a; k += blockDim.x) sIncPtr[k] = A.c.inc_ptr[k];
        // one (a, b) for every pair and no statics (identical agents): the constants live in registers
        bool same = true;
        for (int p = tid; p < np_; p += blockDim.x)
            same = same && A.c.pair_j[p] >= 0 && A.c.pair_a[p] == A.c.pair_a[0] && A.c.pair_b[p] == A.c.pair_b[0];
        uni = __syncthreads_and(same) != 0;
        // incidence entries as scratch byte offsets of the pair's record, bit 0 = negative sign
        for (int k = tid; k < n_inc; k += blockDim.x) {
            const int pe = A.c.inc_pair[k];
            sInc[k] = pe >= 0 ? pe * (kScrW * 8) : (-pe - 1) * (kScrW * 8) + 1;
        }
    }
    double* xg = A.s.xi + (int64_t)i * 3 * nv;
    const double* bg = A.c.b_eq + (int64_t)i * 3 * neq;
    if (init) {
        // straight-line coefficients per agent and axis (solver_multiagent.py:230-235)
        for (int k = tid; k < 3 * nv; k += blockDim.x) {
            const int ax = k / nv, r = k - ax * nv, a = r / m, cc = r - a * m;
            const double p0 = bg[ax * neq + 6 * a + 0], p1 = bg[ax * neq + 6 * a + 3];
            const double v = A.c.line_u[cc] * p0 + A.c.line_v[cc] * (p1 - p0);
            sXi[k] = v;
            xg[k] = v;
        }
    } else if (prime || pre_qp) {
        for (int k = tid; k < 3 * nv; k += blockDim.x) sXi[k] = xg[k];
    } else {
        const double* sg = A.s.sums + (int64_t)i * 2 * n_a * 3 * m;
        for (int k = tid; k < 2 * n_a * 3 * m; k += blockDim.x) sSumIn[k] = sg[k];
        __syncthreads();
        // rhs_k = [ -q_k ; b_eq_k ],  -q = rho B - C  (contracted per agent: [a][k][c])
        for (int k = tid; k < 3 * nk; k += blockDim.x) {
            const int ax = k / nk, r = k - ax * nk;
            double v;
            if (r < nv) {
                const int a = r / m, cc = r - a * m;
                const int o = (a * 3 + ax) * m + cc;
                v = rho * sSumIn[o] - sSumIn[n_a * 3 * m + o];
            } else {
                v = bg[ax * neq + (r - nv)];
            }
            sRhs[k] = v;
        }
        __syncthreads();
        // one warp per row of K^-1 (coalesced, read once for the three axes), shuffle-reduced
        const double* Kl = A.c.kinv + (int64_t)level * nk * nk;
        for (int r = warp; r < nv; r += kMaWarps) {
            const double* Kr = Kl + (int64_t)r * nk;
            double a0 = 0.0, a1 = 0.0, a2 = 0.0;
            for (int q = lane; q < nk; q += 32) {
                const double kv = ld_const(Kr + q);
                a0 = fma(kv, sRhs[q], a0);
                a1 = fma(kv, sRhs[nk + q], a1);
                a2 = fma(kv, sRhs[2 * nk + q], a2);
            }
            a0 = warp_sum(a0);
            a1 = warp_sum(a1);
            a2 = warp_sum(a2);
            if (lane == 0) {
                sXi[r] = a0;
                sXi[nv + r] = a1;
                sXi[2 * nv + r] = a2;
                xg[r] = a0;
                xg[nv + r] = a1;
                xg[2 * nv + r] = a2;
            }
        }
    }
    __syncthreads();
    if (mode == 0 && A.c.bnd) {
        // project every agent's new coefficients onto its boundary conditions, c -= A+ (A c - b) (the explicit
        // K^-1's ~1e-8 there; the reference's LU solve holds them to ~1e-13): one thread per (axis, agent)
        const double* Ab = A.c.bnd;           // 6 x m
        const double* Ap = A.c.bnd + 6 * m;   // m x 6
        for (int k = tid; k < 3 * n_a; k += blockDim.x) {
            const int ax = k / n_a, a = k - ax * n_a;
            double* c = sXi + ax * nv + a * m;
            const double* bv = bg + ax * neq + 6 * a;
            double r[6];
#pragma unroll
            for (int e = 0; e < 6; ++e) {
                double acc = -bv[e];
                for (int cc = 0; cc < m; ++cc) acc = fma(Ab[e * m + cc], c[cc], acc);
                r[e] = acc;
            }
            for (int cc = 0; cc < m; ++cc) {
                double acc = c[cc];
#pragma unroll
                for (int e = 0; e < 6; ++e) acc = fma(-Ap[cc * 6 + e], r[e], acc);
                c[cc] = acc;
                xg[ax * nv + a * m + cc] = acc;
            }
        }
        __syncthreads();
    }
    {
        // coefficients to [c][agent][axis]: the per-round position products read consecutive words
        constexpr int kPer = (3 * 16 * 11 + kMaWarps * 32 - 1) / (kMaWarps * 32);  // n_a <= 16, m <= 11
        double tv[kPer];
#pragma unroll
        for (int j = 0; j < kPer; ++j) {
            const int k = tid + j * kMaWarps * 32;
            tv[j] = k < 3 * nv ? sXi[k] : 0.0;
        }
        __syncthreads();
#pragma unroll
        for (int j = 0; j < kPer; ++j) {
            const int k = tid + j * kMaWarps * 32;
            if (k < 3 * nv) {
                const int ax = k / nv, r = k - ax * nv, a = r / m, cc = r - a * m;
                sXi[cc * 3 * n_a + a * 3 + ax] = tv[j];
            }
        }
        __syncthreads();
    }
    // ---------------- element pass in rounds of kMaWarps samples: warp w takes t = r kMaWarps + w, lanes
    // over pairs; the warp then scatters its pairs' recon / lambda to the agents (fixed incidence order)
    // into V[round parity][w], and after one barrier the CTA contracts the round's V rows with P[t][:] as
    // 8x8x4 fp64 tensor-core tiles (accumulated across rounds in the owning warp's registers).
    const int tasks = 2 * n_a;
    const int rows = tasks * 3;  // [which][agent][axis]
    const int vs = ma_vstride(n_a);  // V row stride: the DMMA A-fragment reads hit 16 distinct bank pairs
    // contraction tiles: D[rows x m] = V^T[rows x t] P[t x m] as 8x8 DMMA tiles, warp w owning tiles
    // w, w + kMaWarps, ... (rows <= 96, m <= 11: at most 12 x 2 tiles, <= 3 per warp)
    constexpr int kMaxTiles = (24 + kMaWarps - 1) / kMaWarps;
    const int n_mt = (rows + 7) >> 3, n_nt = (m + 7) >> 3;
    double cacc[kMaxTiles][2];
#pragma unroll
    for (int j = 0; j < kMaxTiles; ++j) cacc[j][0] = cacc[j][1] = 0.0;
    double sumsq = 0.0, mx = 0.0;
    const int rowW = 3 * np_;  // state[i][t][w][p], W = 3 (a problem's block stays far below 2^31 doubles)
    double* st;  // pinned in a register: rematerialising the 64-bit product per element cost ~20 instructions
    asm volatile("mov.b64 %0, %1;" : "=l"(st) : "l"(A.s.state + (int64_t)i * n_p * rowW));
    const int64_t nplane = (int64_t)A.d.n_problems * n_p * np_;

    const double ir = 1.0 / rho;
    // lambda of this lane's next element, loaded one element ahead (two HBM loads in flight per lane)
    double nlx = 0.0, nly = 0.0, nlz = 0.0;
    if (mode == 0 && warp < n_p && lane < np_) {
        const double* r0 = st + warp * rowW + lane;
        nlx = ld_stream(r0);
        nly = ld_stream(r0 + np_);
        nlz = ld_stream(r0 + 2 * np_);
    }
    const double u_pa = sPair[0], u_pb = sPair[np_], u_ipa = sPair[2 * np_], u_ipb = sPair[3 * np_];
    const double u_pa2 = u_pa * u_pa, u_pb2 = u_pb * u_pb;
    const int n_rounds = (n_p + kMaWarps - 1) / kMaWarps;
    // contraction of round r's samples on the fp64 tensor cores (k = sample within the round), once every
    // warp has published V[r & 1]; then this warp releases the buffer for round r + 2
    auto contract = [&](int r) {
        const int bb = r & 1;
        mbar_wait(&sBar[bb], (uint32_t)((r >> 1) & 1));
        const double* sVb = sV + bb * kMaWarps * vs;
        const int tn = min(kMaWarps, n_p - r * kMaWarps);
        const double* prd = sP + r * kMaWarps * mp;
#pragma unroll
        for (int j = 0; j < kMaxTiles; ++j) {
            const int tile = warp + j * kMaWarps;
            if (tile < n_mt * n_nt) {
                const int mt = tile / n_nt, nt = tile - mt * n_nt;
                const int ar = mt * 8 + (lane >> 2), bc = nt * 8 + (lane >> 2);
#pragma unroll
                for (int ks = 0; ks < (kMaWarps + 3) / 4; ++ks) {
                    const int k = 4 * ks + (lane & 3);
                    const double av = (k < tn && ar < rows) ? sVb[k * vs + ar] : 0.0;
                    const double bv = (k < tn && bc < m) ? prd[k * mp + bc] : 0.0;
                    dmma884(cacc[j], av, bv);
                }
            }
        }
        __syncwarp();
        if (lane == 0) mbar_arrive(&sBar[2 + bb]);
    };
    const bool pf = mode == 0 && lane == 0 && ((rowW * 8) & 15) == 0;
    for (int rd = 0; rd < n_rounds; ++rd) {
        const int t = rd * kMaWarps + warp;
        if (pf && t + kMaAhead * kMaWarps < n_p) prefetch_l2(st + (t + kMaAhead * kMaWarps) * rowW, rowW * 8);
        double* sVr = sV + (rd & 1) * kMaWarps * vs;
        if (t < n_p) {
            // this sample's positions (one (agent, axis) per lane slot; same FMA order as the basis product)
            {
                // slots k0 = lane, k1 = lane + 32 (3 n_a <= 48); lanes past the last slot compute a discarded
                // value from in-bounds shared memory, so the loop is branch-free
                const int xs = 3 * n_a;
                const double* xp = sXi + lane;
                const double* prow = sP + t * mp;
                double p0 = 0.0, p1 = 0.0;
#pragma unroll
                for (int cc = 0; cc < m; ++cc) {
                    const double pv = prow[cc];
                    p0 = fma(pv, xp[0], p0);
                    p1 = fma(pv, xp[32], p1);
                    xp += xs;
                }
                if (lane < xs) sPos[lane] = p0;
                if (lane + 32 < xs) sPos[lane + 32] = p1;
            }
            __syncwarp();
            const double* pt = sPos;
            double* srow = st + t * rowW;
            // the pair pass, specialised on whether the pair constants are uniform (registers, no loads)
            auto pair_pass = [&](auto uni_tag) {
                constexpr bool UNI = decltype(uni_tag)::value;
#pragma unroll kMaPairUnroll
                for (int p = lane; p < np_; p += 32) {
                    double clx = 0.0, cly = 0.0, clz = 0.0;
                    if (mode == 0) {
                        clx = nlx, cly = nly, clz = nlz;
                        const int nxt = p + 32 < np_ ? t * rowW + p + 32 : (t + kMaWarps) * rowW + lane;
                        if (nxt < n_p * rowW) {
                            const double* r2 = st + nxt;
                            nlx = ld_stream(r2);
                            nly = ld_stream(r2 + np_);
                            nlz = ld_stream(r2 + 2 * np_);
                        }
                    }
                    const int pi = sPairI[p], pj = sPairJ[p];
                    double pa, pb, ipa, ipb, pa2, pb2;
                    if constexpr (UNI) {
                        pa = u_pa, pb = u_pb, ipa = u_ipa, ipb = u_ipb, pa2 = u_pa2, pb2 = u_pb2;
                    } else {
                        pa = sPair[p], pb = sPair[np_ + p], ipa = sPair[2 * np_ + p], ipb = sPair[3 * np_ + p];
                        pa2 = pa * pa, pb2 = pb * pb;
                    }
                    double cen[3];
                    if (UNI || pj >= 0) {
    #pragma unroll
                        for (int k = 0; k < 3; ++k) cen[k] = pt[pj * 3 + k];
                    } else {
    #pragma unroll
                        for (int k = 0; k < 3; ++k) cen[k] = sPair[(4 + k) * np_ + p];
                    }
                    const double dx = pt[pi * 3 + 0] - cen[0], dy = pt[pi * 3 + 1] - cen[1], dz = pt[pi * 3 + 2] - cen[2];
                    // alpha = atan2(dy, dx), beta = atan2(hypot(dx/pa, dy/pa), dz/pb) (:280-282)
                    const int64_t ex_i = ((int64_t)i * n_p + t) * np_ + p;
                    auto angles = [&](double& ca, double& sa, double& cb, double& sb) {  // as unit vectors
                        const double h2 = fma(dx, dx, dy * dy);
                        double planar;
                        if (h2 > 0.0) {
                            const double r = rsqrt_fast(h2);
                            ca = dx * r;
                            sa = dy * r;
                            planar = h2 * r * ipa;  // hypot(dx, dy) / pa
                        } else {
                            ca = flip_sign(1.0, sign_bit(dx));
                            sa = flip_sign(0.0, sign_bit(dy));
                            planar = 0.0;
                        }
                        unit2(dz * ipb, planar, &cb, &sb);
                    };
                    double ca = 0.0, sa = 0.0, cb = 0.0, sb = 0.0;
                    double lx, ly, lz, d, rx, ry, rz;
                    if constexpr (!prime && !init) {
                        lx = clx;
                        ly = cly;
                        lz = clz;
                        // The polar update collapsed: with the unit vectors of the offset delta, pa sb ca = dx / g,
                        // pa sb sa = dy / g, pb cb = dz / g and pa^2 sb^2 + pb^2 cb^2 = |delta|^2 / g^2, where
                        // g^2 = (dx^2 + dy^2) / pa^2 + dz^2 / pb^2.  So the multiplier-shifted quadratic (:285-293)
                        // is q = g (delta . (delta + lambda / rho)) / |delta|^2 and the reconstruction is
                        // (d / g) delta: no angle is formed (same quantities up to rounding)
                        const double h2 = fma(dx, dx, dy * dy);
                        const double g2 = fma(dz * dz, ipb * ipb, h2 * (ipa * ipa));
                        if (g2 > 0.0) {
                            const double rg = rsqrt_fast(g2);
                            const double dot = fma(dz, fma(lz, ir, dz), fma(dy, fma(ly, ir, dy), dx * fma(lx, ir, dx)));
                            const double q = dot * (g2 * rg) * rcp_fast(fma(dz, dz, h2));
                            d = q < 1.0 ? 1.0 : (q > 1e6 ? 1e6 : q);
                            const double sc = d * rg;
                            rx = sc * dx;
                            ry = sc * dy;
                            rz = sc * dz;
                        } else {  // delta == 0: atan2's conventions (alpha = 0 / pi, beta = 0 / pi along z)
                            angles(ca, sa, cb, sb);
                            const double q = pb * cb * fma(lz, ir, dz) * rcp_fast(pb2);
                            d = q < 1.0 ? 1.0 : (q > 1e6 ? 1e6 : q);
                            rx = pa * d * sb * ca;
                            ry = pa * d * sb * sa;
                            rz = pb * d * cb;
                        }
                        if (A.s.export_d) angles(ca, sa, cb, sb);  // the exported angles
                    } else {
                        if (prime) {  // the given state's angles
                            sincos(A.s.export_ab[ex_i], &sa, &ca);
                            sincos(A.s.export_ab[nplane + ex_i], &sb, &cb);
                            lx = srow[p];
                            ly = srow[np_ + p];
                            lz = srow[2 * np_ + p];
                            d = A.s.export_d[ex_i];
                        } else {  // init
                            angles(ca, sa, cb, sb);
                            lx = ly = lz = 0.0;
                            d = 1.0;
                        }
                        rx = pa * d * sb * ca;
                        ry = pa * d * sb * sa;
                        rz = pb * d * cb;
                    }
                    (void)pa2;
                    if (prime) {
                    } else if (!init) {
                        const double ex = dx - rx, ey = dy - ry, ez = dz - rz;  // residual (:203-208)
                        sumsq = fma(ex, ex, fma(ey, ey, fma(ez, ez, sumsq)));
                        const double ae = fabs(ex) > fabs(ey) ? fabs(ex) : fabs(ey);
                        const double am = ae > fabs(ez) ? ae : fabs(ez);
                        mx = am > mx ? am : mx;
                        lx = fma(rho, ex, lx);  // lambda += rho * res (:296)
                        ly = fma(rho, ey, ly);
                        lz = fma(rho, ez, lz);
                        st_stream(srow + p, lx);
                        st_stream(srow + np_ + p, ly);
                        st_stream(srow + 2 * np_ + p, lz);
                    } else {
                        srow[p] = 0.0;
                        srow[np_ + p] = 0.0;
                        srow[2 * np_ + p] = 0.0;
                    }
                    if (!prime && A.s.export_d) {  // runtime: batch and single solves share one code path
                        const int64_t e = ex_i;
                        A.s.export_d[e] = d;
                        A.s.export_ab[e] = atan2(sa, ca);           // the reference's stored angles
                        A.s.export_ab[nplane + e] = atan2(sb, cb);
                    }
                    // next RHS: recon (+ static centre) and lambda, scattered to the pair's agents below
                    double* sc = sScr + p * kScrW;
                    sc[0] = rx + (pj < 0 ? cen[0] : 0.0);
                    sc[1] = ry + (pj < 0 ? cen[1] : 0.0);
                    sc[2] = rz + (pj < 0 ? cen[2] : 0.0);
                    sc[3] = lx;
                    sc[4] = ly;
                    sc[5] = lz;
                }
            };
            if (uni)
                pair_pass(std::integral_constant<bool, true>{});
            else
                pair_pass(std::integral_constant<bool, false>{});
            __syncwarp();
            // per-agent signed incidence sums (fixed order) -> V[w][which][agent][axis]; V[rd & 1] was last
            // read by round rd - 2's contraction
            if (rd >= 2) mbar_wait(&sBar[2 + (rd & 1)], (uint32_t)(((rd - 2) >> 1) & 1));
            for (int task = lane; task < tasks; task += 32) {
                const int a = task % n_a, which = task / n_a;  // which 0: B (recon), 1: C (lambda)
                double v[3] = {0.0, 0.0, 0.0};
                const char* base = reinterpret_cast<const char*>(sScr + 3 * which);
                for (int q = sIncPtr[a]; q < sIncPtr[a + 1]; ++q) {
                    const int w = sInc[q];
                    const double sgn = (w & 1) ? -1.0 : 1.0;
                    const double* sc = reinterpret_cast<const double*>(base + (w & ~7));
#pragma unroll
                    for (int k = 0; k < 3; ++k) v[k] = fma(sgn, sc[k], v[k]);
                }
                double* vo = sVr + warp * vs + task * 3;
                vo[0] = v[0];
                vo[1] = v[1];
                vo[2] = v[2];
            }
        }
        // V[b] complete for this warp: publish it, then contract the previous round (usually already
        // published by every warp, so no CTA-wide barrier per round)
        __syncwarp();
        if (lane == 0) mbar_arrive(&sBar[rd & 1]);
        if (rd > 0) contract(rd - 1);
    }
    contract(n_rounds - 1);

    // ---------------- reductions
    sumsq = warp_sum(sumsq);
    mx = warp_max(mx);
    if (lane == 0) {
        sWarp[warp] = sumsq;
        sWarp[kMaWarps + warp] = mx;
    }
    double* sg = A.s.sums + (int64_t)i * 2 * n_a * 3 * m;  // [which][a][k][c] = [row][c]
#pragma unroll
    for (int j = 0; j < kMaxTiles; ++j) {
        const int tile = warp + j * kMaWarps;
        if (tile < n_mt * n_nt) {
            const int mt = tile / n_nt, nt = tile - mt * n_nt;
            const int r = mt * 8 + (lane >> 2), c0 = nt * 8 + 2 * (lane & 3);
            if (r < rows) {
                if (c0 < m) sg[r * m + c0] = cacc[j][0];
                if (c0 + 1 < m) sg[r * m + c0 + 1] = cacc[j][1];
            }
        }
    }
    __syncthreads();
    if (tid == 0 && mode == 0) {
        double ss = 0.0, mm = 0.0;
        for (int w = 0; w < kMaWarps; ++w) {
            ss += sWarp[w];
            mm = fmax(mm, sWarp[kMaWarps + w]);
        }
        if (ss != ss) mm = ss;
        const double nrm = sqrt(ss);
        A.s.res_norm[i] = nrm;
        A.s.res_max[i] = mm;
        const int it = A.s.iteration[i] + 1;  // _iterate: state.iteration += 1
        A.s.iteration[i] = it;
        const int nh = A.s.n_hist[i];
        if (A.s.hist && nh < A.p.max_hist) {
            double* h = A.s.hist + ((int64_t)i * A.p.max_hist + nh) * 3;
            h[0] = nrm;
            h[1] = mm;
            h[2] = rho;
        }
        const int n = nh + 1;
        A.s.n_hist[i] = n;
        const int w = A.p.stall_window, w2 = 2 * w;
        double* ring = A.s.ring + (int64_t)i * w2;
        ring[(n - 1) % w2] = nrm;
        if (nrm <= A.p.tol_norm) {  // solver_multiagent.py:319-321
            A.s.status[i] = status0 | TRO_CONVERGED;
        } else {
            const int nl = A.d.n_levels;
            const int mi = A.p.max_iter > 1 ? A.p.max_iter : 1;
            int scheduled = (int)((double)it * nl / (double)mi);  // :325
            if (scheduled > nl - 1) scheduled = nl - 1;
            bool stalled = false;
            const int lc = A.s.last_change[i];
            if (n >= w2 && it - lc >= w) {  // :327-331 (np.mean in numpy's summation order)
                const double recent = np_mean_ring(ring, n - w, w, w2), previous = np_mean_ring(ring, n - w2, w, w2);
                stalled = previous > 0.0 && (previous - recent) / previous < A.p.stall_improvement;
            }
            const int target = scheduled > (stalled ? level + 1 : level) ? scheduled : (stalled ? level + 1 : level);
            if (target > level && level < nl - 1) {  // :332-335
                A.s.level[i] = target < nl - 1 ? target : nl - 1;
                A.s.last_change[i] = it;
            }
        }
    }
}

// ---------------------------------------------------------------- batched QP step on the fp64 tensor cores
// xi_i = K_L^-1 [ rho B_i - C_i ; b_eq_i ] for every axis of every non-converged problem, as one GEMM per
// CTA: D[nv x 3P] = K_L^-1[0:nv, 0:nk] x R[nk x 3P] with DMMA (mma.sync m8n8k4 f64), P = 8 problems.
// The fused kernel's per-problem GEMV reads the nv x nk inverse once per problem (~36 k instructions per
// problem); here a CTA reads it once for 8 problems and the tensor cores do the FMAs.  Problems of a tile
// at different rho levels are handled level by level (the schedule keeps them together almost always).
constexpr int kQpP = 8;                // problems per CTA (16: 117 us, 8: 87 us, 4: 116 us at C3)
constexpr int kQpCols = 3 * kQpP;      // 48 RHS columns
constexpr int kQpLd = kQpCols + 4;     // padded smem row (bank spread of the B fragments)
constexpr int kQpMt = 3;               // m-tiles per warp (8 warps x 3 x 8 rows >= nv = 176)


template <int M>
__global__ void __launch_bounds__(256) ma_qp_kernel(MaArgs A) {
    extern __shared__ double smem[];
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int n_a = A.d.n_agents, neq = A.d.n_eq;
    constexpr int m = M;
    const int nv = n_a * m, nk = nv + neq, nk4 = (nk + 3) & ~3;
    const int i0 = blockIdx.x * kQpP;
    const int npb = min(kQpP, A.d.n_problems - i0);
    double* sR = smem;                          // [nk4][kQpLd]
    int* sLev = reinterpret_cast<int*>(smem + nk4 * kQpLd);  // [kQpP] level, -1: skip
    if (tid < kQpP) {
        int lv = -1;
        if (tid < npb && !(A.s.status[i0 + tid] & TRO_CONVERGED)) lv = A.s.level[i0 + tid];
        sLev[tid] = lv;
    }
    __syncthreads();
    // RHS columns (problem p, axis ax) = [ rho B - C ; b_eq ]  (agent sums [which][a][k][c])
    for (int e = tid; e < nk4 * kQpCols; e += blockDim.x) {
        const int r = e / kQpCols, col = e - r * kQpCols;
        const int p = col / 3, ax = col - 3 * p;
        double v = 0.0;
        const int lv = sLev[p];
        if (lv >= 0 && r < nk) {
            const int i = i0 + p;
            if (r < nv) {
                const int a = r / m, cc = r - a * m;
                const double* sg = A.s.sums + (int64_t)i * 2 * n_a * 3 * m;
                const int o = (a * 3 + ax) * m + cc;
                v = A.c.level_rho[lv] * sg[o] - sg[n_a * 3 * m + o];
            } else {
                v = A.c.b_eq[(int64_t)i * 3 * neq + ax * neq + (r - nv)];
            }
        }
        sR[r * kQpLd + col] = v;
    }
    __syncthreads();
    const int arow = lane >> 2, acol = lane & 3;  // A fragment: A[row][k]; B fragment: B[k = lane & 3][col = lane >> 2]
    for (int pass = 0; pass < kQpP; ++pass) {
        // the level of this pass: the first not-yet-done problem's (uniform across the CTA)
        int lv = -1;
        for (int p = 0; p < kQpP; ++p) {
            if (sLev[p] >= 0) {
                lv = sLev[p];
                break;
            }
        }
        if (lv < 0) break;
        const double* K = A.c.kinv + (int64_t)lv * nk * nk;
        double acc[kQpMt][kQpCols / 8][2];
#pragma unroll
        for (int t = 0; t < kQpMt; ++t)
#pragma unroll
            for (int n = 0; n < kQpCols / 8; ++n) acc[t][n][0] = acc[t][n][1] = 0.0;
        // A fragments (K^-1 from L2) loaded kPre k-steps ahead: a k-step's 18 DMMA do not cover an L2 load
        constexpr int kPre = MA_QP_PRE;
        auto load_a = [&](int k0, double* af) {
            const int kk = k0 + acol;
#pragma unroll
            for (int t = 0; t < kQpMt; ++t) {
                const int row = (warp + 8 * t) * 8 + arow;
                af[t] = (row < nv && kk < nk) ? ld_const(K + (int64_t)row * nk + kk) : 0.0;
            }
        };
        double ring[kPre][kQpMt];
#pragma unroll
        for (int u = 0; u < kPre; ++u) load_a(4 * u, ring[u]);
        for (int k0 = 0; k0 < nk4; k0 += 4 * kPre) {
#pragma unroll
            for (int u = 0; u < kPre; ++u) {
                const int kc = k0 + 4 * u;
                if (kc >= nk4) break;
                double af[kQpMt];
#pragma unroll
                for (int t = 0; t < kQpMt; ++t) af[t] = ring[u][t];
                load_a(kc + 4 * kPre, ring[u]);  // rows beyond nk read as zero
#pragma unroll
                for (int n = 0; n < kQpCols / 8; ++n) {
                    const double bf = sR[(kc + acol) * kQpLd + n * 8 + arow];
#pragma unroll
                    for (int t = 0; t < kQpMt; ++t) dmma884(acc[t][n], af[t], bf);
                }
            }
        }
        // D fragment: rows (mtile * 8 + lane >> 2), columns n * 8 + 2 (lane & 3) + {0, 1}
#pragma unroll
        for (int t = 0; t < kQpMt; ++t) {
            const int row = (warp + 8 * t) * 8 + arow;
            if (row >= nv) continue;
#pragma unroll
            for (int n = 0; n < kQpCols / 8; ++n)
#pragma unroll
                for (int h = 0; h < 2; ++h) {
                    const int col = n * 8 + 2 * acol + h;
                    const int p = col / 3, ax = col - 3 * p;
                    if (sLev[p] == lv) A.s.xi[(int64_t)(i0 + p) * 3 * nv + ax * nv + row] = acc[t][n][h];
                }
        }
        __syncthreads();
        if (tid < kQpP && sLev[tid] == lv) sLev[tid] = -1;  // done
        __syncthreads();
    }
}

template <int M, int MODE>
static int ma_launch(const MaArgs& A, size_t smem, cudaStream_t st) {
    cudaFuncSetAttribute(ma_kernel<M, MODE>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    ma_kernel<M, MODE><<<A.d.n_problems, kMaWarps * 32, smem, st>>>(A);
    return (int)cudaGetLastError();
}

template <int M>
static int ma_dispatch_m(const MaArgs& A, int mode, bool, size_t smem, cudaStream_t st) {
    if (mode == 0) return ma_launch<M, 0>(A, smem, st);
    if (mode == 1) return ma_launch<M, 1>(A, smem, st);
    if (mode == 4) return ma_launch<M, 4>(A, smem, st);
    if (mode == 3) {
        const int nk = A.d.n_agents * M + A.d.n_eq, nk4 = (nk + 3) & ~3;
        const size_t qsm = (size_t)nk4 * kQpLd * sizeof(double) + kQpP * sizeof(int);
        if (qsm > 227 * 1024 || A.d.n_agents * M > 8 * kQpMt * 8) return TRO_EINVAL;
        cudaFuncSetAttribute(ma_qp_kernel<M>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)qsm);
        ma_qp_kernel<M><<<(A.d.n_problems + kQpP - 1) / kQpP, 256, qsm, st>>>(A);
        return (int)cudaGetLastError();
    }
    return ma_launch<M, 2>(A, smem, st);
}

static int ma_dispatch(const MaArgs& A, int mode, bool exp, size_t smem, cudaStream_t st) {
    return A.d.m == 11 ? ma_dispatch_m<11>(A, mode, exp, smem, st) : ma_dispatch_m<9>(A, mode, exp, smem, st);
}

}  // namespace tro

extern "C" int tro_ma_run(int32_t mode, const tro_ma_dims* d, const tro_ma_consts* c, const tro_ma_state* s,
                          const tro_ma_params* p, void* stream) {
    if (!d || !c || !s || !p || mode < 0 || mode > 4) return TRO_EINVAL;
    if (mode == 1 && (!s->export_d || !s->export_ab)) return TRO_EINVAL;
    if (d->n_agents < 1 || d->n_agents > tro::kMaMaxAgents || d->n_p < 2 || d->m < 1 || d->n_pairs < 1 ||
        d->n_levels < 1 || p->stall_window < 1 || 2 * p->stall_window > tro::kMaMaxRing)
        return TRO_EINVAL;
    if (d->m != 11 && d->m != 9) return TRO_EINVAL;  // per-lane register accumulators are compile-time sized
    if (2 * d->n_agents > 32) return TRO_EINVAL;
    if (d->n_problems <= 0) return 0;
    tro::MaArgs A;
    A.d = *d;
    A.c = *c;
    A.s = *s;
    A.p = *p;
    // every pair appears in at most two agent incidence lists
    const tro::MaSmem L = tro::ma_layout(d->n_p, d->m, d->n_agents, d->n_pairs, d->n_eq, 2 * d->n_pairs);
    const size_t smem = (size_t)L.total * sizeof(double);
    if (smem > 227 * 1024) return TRO_EINVAL;
    cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
    const bool exp = s->export_d != nullptr && s->export_ab != nullptr;
    return tro::ma_dispatch(A, mode, exp, smem, st);
}
