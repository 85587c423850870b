// Batched 2-D footprint + heading AM iteration (arXiv 2408.10731, Alg. 2) for sm_100a.
//
// One CTA owns one batch member for one batch_iteration (solver_batch.py:352-363):
//   prologue : xi = K_xi^-1 [-(q - lam - rho F'g) ; b] from the F'g sums the previous launch
//              left behind (batch_xi_step, :292-299); F is never materialised;
//   heading  : per sample, the copies' angle atan2(s, c), nearest-branch unwrapped against the
//              previous heading (:308-310), contracted with P and pushed through K_psi^-1
//              (:311-314);
//   body     : per sample t (one thread), velocity / acceleration rows and every
//              (circle, obstacle) element: footprint offset (:196-204), alpha_coll as a unit
//              vector (atan2 is never needed: only its cos / sin enter, :318-326), the clipped
//              scale d (:329-344), targets g (:207-227), residual F xi - g (:347-349);
//   epilogue : per-sample partial sums contracted with P / Pdot / Pddot in a fixed order into
//              F'g (next launch's RHS) and F'r (multiplier ascent, :359), the heading
//              multiplier (:360-361), per-member max |r| and ||r||; the last CTA to finish reduces
//              the batch (argmin of ||r||, min of max |r|, :454-460) and applies the
//              batch-global stall rule (_maybe_grow_rho, :396-406).
// alpha / d are never stored: they are pure functions of (xi, heading) and only feed F'g.
#include "common.cuh"
#include "fastmath.cuh"
#include "../../include/trajopt_b200.h"

namespace tro {

// np.clip semantics (NaN passes through) in 2 compares + selects; fmin / fmax cost 4 SASS each
__device__ __forceinline__ double clip(double x, double lo, double hi) { return x < lo ? lo : (x > hi ? hi : x); }
__device__ __forceinline__ double dmax(double a, double b) { return a > b ? a : b; }

constexpr int kB2Threads = 128;
#ifndef B2_Q
#define B2_Q 8  // t-chunks of the F' contraction (partials in shared memory)
#endif
constexpr int kB2Q = B2_Q;
constexpr int kB2Warps = kB2Threads / 32;
constexpr int kB2MaxRing = 64;
constexpr int kB2MaxC = 8;
constexpr int kB2MaxM = 16;
#ifndef B2_UNROLL_BASIS
#define B2_UNROLL_BASIS 4  // unroll count of the per-sample basis products (C2-alt: 1 -> 45.1, 2 -> 44.2, 4 -> 44.0, 8 -> 53.3, 16 -> 45.5 us/it)
#endif
#ifndef B2_OBS_BATCH
#define B2_OBS_BATCH 5  // obstacles whose track loads are issued before the first use (element pass; 8 spilled more: 49.8 vs 47.0 us per C2-alt iteration)
#endif
#ifndef B2_MINB
#define B2_MINB 7  // 7 CTAs / SM (72 registers, some spills): C2-alt's 1024 members in one wave; 6 % faster than 4 CTAs / 128 registers at 1024 and 8192 members (tools/tune_b2.sh)
#endif
constexpr int kB2UnrollM = B2_UNROLL_BASIS > 0 ? B2_UNROLL_BASIS : 1;

struct B2Args {
    tro_b2_dims d;
    tro_b2_consts c;
    tro_b2_state s;
    tro_b2_params p;
};

// per-sample shared arrays
// The F'g rows reuse the geometry rows kX..kAY: a sample's thread reads its geometry into registers before
// it writes that sample's F'g inputs, and no other thread reads them (18 rows instead of 26: the smaller
// per-CTA footprint leaves L1 room for the shared obstacle tracks and basis rows at 7 CTAs / SM).
enum {
    kX, kY, kC, kS, kVX, kVY, kAX, kAY, kTgt,                // geometry of the new xi
    kRVX, kRVY, kRAX, kRAY, kRX, kRY, kRCX, kRCY, kDPsi,    // F'r / heading residual inputs
    kNT,
    kGVX = kX, kGVY, kGAX, kGAY, kGX, kGY, kGCX, kGCY,      // F'g inputs (aliasing the geometry rows)
};
static_assert(kGCY < kTgt, "the F'g rows must not overlap the heading targets");

struct B2Smem {
    int T, xi, rhs, po, pn, rp, out, part, ab, ai, red, total;
};
__host__ __device__ inline B2Smem b2_layout(int n_p, int m, int n_o) {
    B2Smem L;
    const int nv = 4 * m, nk = nv + 12;
    int off = 0;
    L.T = off;    off += kNT * n_p;
    L.xi = off;   off += nv;
    L.rhs = off;  off += nk;
    L.po = off;   off += m;
    L.pn = off;   off += m;
    L.rp = off;   off += m + 2;
    L.out = off;  off += 2 * nv + m;
    L.part = off; off += kB2Q * (2 * nv + m);
    L.ab = off;   off += 5 * (n_o > 0 ? n_o : 1);  // per obstacle (a, b, a^2, b^2, 1/a)
    off = (off + 1) & ~1;
    L.ai = off;   off += 2 * (n_o > 0 ? n_o : 1);  // per obstacle (a^2, (1e6 a)^2), 16-byte aligned
    L.red = off;  off += 2 * kB2Warps + 2;
    L.total = off;
    return L;
}

// One (circle, obstacle, sample) element: alpha_coll = atan2(dy, dx) (:324), the clipped scale
// (:338-340) and the target offset (ex, ey) = (a d cos alpha, b d sin alpha) (:221-222).
// Circles (a == b) use d = clip(h / a) and (ex, ey) = (dx, dy) a d / h: the same quantities without
// the num / den quotient (the reference's num / den equals h / a up to rounding).
__device__ __forceinline__ void b2_element(double dx, double dy, const double* ab, bool circle, double* ex,
                                           double* ey, double* dout) {
    const double a = ab[0];
    const double h2 = fma(dx, dx, dy * dy);
    if (circle && h2 > 0.0) {
        const double r = rsqrt_fast(h2);
        const double d = clip(h2 * r * ab[4], 1.0, 1.0e6);  // ab[4]: 1 / a
        const double s = a * d * r;
        *ex = dx * s;
        *ey = dy * s;
        *dout = d;
        return;
    }
    const double b = ab[1];
    double ca, sa;
    unit2(dx, dy, &ca, &sa);
    const double num = a * dx * ca + b * dy * sa;
    const double den = ab[2] * (ca * ca) + ab[3] * (sa * sa);
    const double d = clip(num * rcp_fast(den), 1.0, 1.0e6);
    *ex = a * d * ca;
    *ey = b * d * sa;
    *dout = d;
}


// Batch bookkeeping of one iteration (solver_batch.py:454-461): the best member (argmin of the
// residual norm, first index on ties; numpy's argmin returns the first NaN if there is one), its
// max |r|, and the batch minimum of max |r|.  A "summary" is (best norm, best global index, its max,
// min max); shard summaries merge associatively, so a sharded batch (TRO_B2_SHARD + mode 6) makes
// exactly the single-GPU decisions.
struct B2Summary {
    double best, best_max, mmin;
    int64_t bidx;   // global member index, -1: none
    bool nan_norm;  // best is the first NaN norm
    bool nan_max;   // some max |r| is NaN
};

__device__ __forceinline__ bool b2_better(double nb, int64_t ni, bool nn, double ob, int64_t oi, bool on) {
    if (ni < 0) return false;
    if (oi < 0) return true;
    if (nn != on) return nn;       // NaN beats numbers
    if (nn) return ni < oi;        // first NaN
    return nb < ob || (nb == ob && ni < oi);
}

__device__ B2Summary b2_warp_merge(B2Summary v) {
    for (int o = 16; o > 0; o >>= 1) {
        const double ob = __shfl_xor_sync(0xffffffffu, v.best, o);
        const double om = __shfl_xor_sync(0xffffffffu, v.best_max, o);
        const long long oi = __shfl_xor_sync(0xffffffffu, (long long)v.bidx, o);
        const bool on = __shfl_xor_sync(0xffffffffu, (int)v.nan_norm, o) != 0;
        if (b2_better(ob, oi, on, v.best, v.bidx, v.nan_norm)) v.best = ob, v.best_max = om, v.bidx = oi, v.nan_norm = on;
        v.mmin = fmin(v.mmin, __shfl_xor_sync(0xffffffffu, v.mmin, o));
    }
    v.nan_max = __any_sync(0xffffffffu, v.nan_max);
    return v;
}

// warp 0 of the last CTA: summary of this launch's members (global index = offset + k)
__device__ B2Summary b2_member_summary(const B2Args& A) {
    const int lane = threadIdx.x & 31;
    const int64_t B = A.d.n_members, off = A.p.member_offset;
    B2Summary v{__longlong_as_double(0x7ff0000000000000LL), 0.0, __longlong_as_double(0x7ff0000000000000LL), -1,
                false, false};
    // this tail runs in one warp after every other CTA finished: keep 16 L2 loads in flight per lane
    constexpr int kLd = 16;
    for (int64_t base = 0; base < B; base += 32 * kLd) {
        double nv[kLd], mv[kLd];
#pragma unroll
        for (int j = 0; j < kLd; ++j) {
            const int64_t k = base + j * 32 + lane;
            nv[j] = k < B ? __ldcg(A.s.res_norm + k) : 0.0;
            mv[j] = k < B ? __ldcg(A.s.res_max + k) : 0.0;
        }
#pragma unroll
        for (int j = 0; j < kLd; ++j) {
            const int64_t k = base + j * 32 + lane;
            if (k >= B) break;
            const bool nn = nv[j] != nv[j];
            if (b2_better(nv[j], off + k, nn, v.best, v.bidx, v.nan_norm))
                v.best = nv[j], v.best_max = mv[j], v.bidx = off + k, v.nan_norm = nn;
            if (mv[j] != mv[j]) v.nan_max = true;
            else v.mmin = fmin(v.mmin, mv[j]);
        }
    }
    return b2_warp_merge(v);
}

// history row + stall rule (_maybe_grow_rho, :396-406); lane 0 only
__device__ void b2_schedule(const B2Args& A, int level, double rho, const B2Summary& v) {
    const double qnan = __longlong_as_double(0x7ff8000000000000LL);
    const double mmin = v.nan_max ? qnan : v.mmin;
    const int it = A.s.iteration[0] + 1;  // batch_iteration: state.iteration += 1 (:362)
    A.s.iteration[0] = it;
    const int nh = A.s.n_hist[0];
    if (A.s.hist && nh < A.d.max_hist) {
        double* h = A.s.hist + (int64_t)nh * 4;
        h[0] = v.best;
        h[1] = v.best_max;
        h[2] = rho;
        h[3] = (double)v.bidx;
    }
    const int n = nh + 1;
    A.s.n_hist[0] = n;
    const int w = A.p.stall_window, w2 = 2 * w;
    A.s.ring[(n - 1) % w2] = mmin;
    if (A.p.flags & TRO_FLAG_NO_SCHEDULE) return;
    const int lc = A.s.last_change[0];
    if (n >= w2 && it - lc >= w) {  // :398
        // np.mean(history[-w:]), np.mean(history[-2w:-w]) in numpy's summation order
        const double recent = np_mean_ring(A.s.ring, n - w, w, w2), previous = np_mean_ring(A.s.ring, n - w2, w, w2);
        if (previous > fmax(A.p.tol, 0.0) && (previous - recent) / previous < A.p.stall_improvement) {
            if (level + 1 < A.d.n_levels) {
                A.s.level[0] = level + 1;
                A.s.n_changes[0] += 1;
            }
            A.s.last_change[0] = it;  // rho = min(rho * growth, cap): the chain saturates at the cap
        }
    }
}

// last CTA, warp 0: single-GPU bookkeeping, or (TRO_B2_SHARD) this shard's summary for the all-gather
__device__ void b2_batch_epilogue(const B2Args& A, int level, double rho) {
    const B2Summary v = b2_member_summary(A);
    if ((threadIdx.x & 31) != 0) return;
    if (A.p.flags & TRO_B2_SHARD) {
        double* o = A.s.shard;
        o[0] = v.best;
        o[1] = (double)v.bidx;
        o[2] = v.best_max;
        o[3] = v.nan_max ? __longlong_as_double(0x7ff8000000000000LL) : v.mmin;
        return;
    }
    b2_schedule(A, level, rho, v);
}

// mode 6: merge the all-gathered shard summaries (n_shards x 4, rank order) and run the schedule
__global__ void __launch_bounds__(32) b2_merge_kernel(B2Args A) {
    const int lane = threadIdx.x;
    B2Summary v{__longlong_as_double(0x7ff0000000000000LL), 0.0, __longlong_as_double(0x7ff0000000000000LL), -1,
                false, false};
    for (int r = lane; r < A.p.n_shards; r += 32) {
        const double* s = A.s.shards_in + 4 * r;
        const int64_t idx = (int64_t)s[1];
        const bool nn = s[0] != s[0];
        if (idx >= 0 && b2_better(s[0], idx, nn, v.best, v.bidx, v.nan_norm))
            v.best = s[0], v.bidx = idx, v.best_max = s[2], v.nan_norm = nn;
        if (s[3] != s[3]) v.nan_max = true;
        else v.mmin = fmin(v.mmin, s[3]);
    }
    v = b2_warp_merge(v);
    if (lane != 0) return;
    const int level = *A.s.level;
    b2_schedule(A, level, A.c.rho_chain[level], v);
}

enum { kModeIter = 0, kModePrime = 1, kModeMaterialise = 2, kModeRank = 3, kModeXi = 4, kModeHeading = 5 };

// sum_j M[j * ld + col] * v[j] over j < n (v in shared memory), four independent FMA chains
__device__ __forceinline__ double b2_gemv_col(const double* M, int ld, int col, const double* v, int n) {
    const double* p = M + col;
    double a0 = 0.0, a1 = 0.0, a2 = 0.0, a3 = 0.0;
    int j = 0;
    for (; j + 4 <= n; j += 4) {
        a0 = fma(__ldg(p + (int64_t)j * ld), v[j], a0);
        a1 = fma(__ldg(p + (int64_t)(j + 1) * ld), v[j + 1], a1);
        a2 = fma(__ldg(p + (int64_t)(j + 2) * ld), v[j + 2], a2);
        a3 = fma(__ldg(p + (int64_t)(j + 3) * ld), v[j + 3], a3);
    }
    for (; j < n; ++j) a0 = fma(__ldg(p + (int64_t)j * ld), v[j], a0);
    return (a0 + a1) + (a2 + a3);
}

template <int NC, int MODE, bool CIRC>
__global__ void __launch_bounds__(kB2Threads, B2_MINB) b2_kernel(B2Args A) {
    constexpr bool iter = MODE == kModeIter;
    constexpr bool qp_xi = MODE == kModeIter || MODE == kModeXi;
    constexpr bool heading = MODE == kModeIter || MODE == kModeHeading;
    constexpr bool body = MODE <= kModeRank;
    extern __shared__ double smem[];
    const int64_t i = blockIdx.x;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int n_p = A.d.n_p, m = A.d.m, nv = 4 * m, nk = nv + 12;
    const int n_o = A.d.n_obs, n_c = NC ? NC : A.d.n_c;
    const int flags = A.p.flags;
    const bool psi_in = (flags & TRO_B2_PSI_IN) != 0;
    const bool given_alpha = (MODE == kModePrime || MODE == kModeMaterialise || MODE == kModeRank) &&
                             (flags & (TRO_B2_GIVEN_ALPHA | TRO_B2_GIVEN_AD)) != 0;
    const bool given_d = (MODE == kModePrime || MODE == kModeRank) && (flags & TRO_B2_GIVEN_AD) != 0;
    const B2Smem L = b2_layout(n_p, m, n_o);
    double* sT = smem + L.T;
    double* sPart = smem + L.part;
    double* sAB = smem + L.ab;
    double* sAI = smem + L.ai;
    double* sXi = smem + L.xi;
    double* sRhs = smem + L.rhs;
    double* sPo = smem + L.po;
    double* sPn = smem + L.pn;
    double* sRp = smem + L.rp;
    double* sOut = smem + L.out;
    double* sRed = smem + L.red;

    const int level = *A.s.level;
    const double rho = A.c.rho_chain[level], rho_p = A.c.rho_psi_chain[level];
    const double* PT = A.c.PT;
    const double* PdT = PT + (int64_t)m * n_p;
    const double* PddT = PdT + (int64_t)m * n_p;
    const double* Pr = A.c.Pr;
    const double* Pdr = Pr + (int64_t)n_p * m;
    const double* Pddr = Pdr + (int64_t)n_p * m;
    double* g_xi = A.s.xi + i * nv;
    double* g_lam = A.s.lam + i * nv;
    double* g_sum = A.s.sums + i * nv;
    double* g_xp = A.s.xi_psi + i * m;
    double* g_lp = A.s.lam_psi + i * m;
    double* g_psi = A.s.psi ? A.s.psi + i * n_p : nullptr;

    if (body)
        for (int o = tid; o < n_o; o += kB2Threads) {
            const double a = __ldg(A.c.obs_ab + 2 * o), b = __ldg(A.c.obs_ab + 2 * o + 1);
            sAB[5 * o + 0] = a;
            sAB[5 * o + 1] = b;
            sAB[5 * o + 2] = a * a;
            sAB[5 * o + 3] = b * b;
            sAB[5 * o + 4] = 1.0 / a;
            sAI[2 * o] = a * a;                        // clamp-inactive band h^2 in [a^2, (1e6 a)^2]
            sAI[2 * o + 1] = (1.0e6 * a) * (1.0e6 * a);
        }

    // ---------------- prologue: the xi-step QP (batch_xi_step, :292-299) or the current iterate
    if (qp_xi) {
        if (tid < nv) {
            const double ql = (A.c.q[tid] - g_lam[tid]) - rho * g_sum[tid];  // q_lin (:297)
            sRhs[tid] = -ql;                                                   // [-q ; b] (qpcore.py:141)
        } else if (tid < nk) {
            sRhs[tid] = A.c.b[tid - nv];
        }
        __syncthreads();
        // [xi; nu] = K^-1 [-q; b] (qpcore.py:141-143), then one step of iterative refinement:
        // r = rhs - K [xi; nu], xi += (K^-1 r)[:4m].  The explicit inverse alone leaves xi ~1e-11 from the
        // LU solve; the refined xi sits at the LU solve's rounding floor.
        double* sSol = smem + L.part;  // the contraction partials' space is free during the prologue
        double* sRes = sSol + nk;
        const double* Ki = A.c.kinvT_xi + (int64_t)level * nk * nk;
        if (tid < nk) sSol[tid] = b2_gemv_col(Ki, nk, tid, sRhs, nk);
        __syncthreads();
        if (tid < nk)  // K is symmetric: its column tid is row tid, read coalesced across threads
            sRes[tid] = sRhs[tid] - b2_gemv_col(A.c.k_xi + (int64_t)level * nk * nk, nk, tid, sSol, nk);
        __syncthreads();
        if (tid < nv) {
            const double acc = sSol[tid] + b2_gemv_col(Ki, nk, tid, sRes, nk);
            sXi[tid] = acc;
            if (MODE == kModeXi) g_xi[tid] = acc;
        }
        if (MODE == kModeXi) return;
    } else {
        if (tid < nv) sXi[tid] = g_xi[tid];
    }
    if (tid < m) (heading ? sPo : sPn)[tid] = g_xp[tid];
    __syncthreads();

    // ---------------- per-sample geometry of xi; heading targets (heading_step, :307-310)
    for (int t = tid; t < n_p; t += kB2Threads) {
        double x = 0, y = 0, c = 0, s = 0, vx = 0, vy = 0, ax = 0, ay = 0, po = 0;
#pragma unroll kB2UnrollM
        for (int k = 0; k < kB2MaxM; ++k) {  // fully unrolled + predicated: all basis loads in flight at once
            if (k >= m) break;
            const double p = __ldg(PT + k * n_p + t), pd = __ldg(PdT + k * n_p + t), pdd = __ldg(PddT + k * n_p + t);
            x = fma(p, sXi[k], x);
            c = fma(p, sXi[m + k], c);
            y = fma(p, sXi[2 * m + k], y);
            s = fma(p, sXi[3 * m + k], s);
            vx = fma(pd, sXi[k], vx);
            vy = fma(pd, sXi[2 * m + k], vy);
            ax = fma(pdd, sXi[k], ax);
            ay = fma(pdd, sXi[2 * m + k], ay);
            if (heading) po = fma(p, sPo[k], po);
        }
        double* T = sT + t;
        T[kX * n_p] = x;
        T[kY * n_p] = y;
        T[kC * n_p] = c;
        T[kS * n_p] = s;
        T[kVX * n_p] = vx;
        T[kVY * n_p] = vy;
        T[kAX * n_p] = ax;
        T[kAY * n_p] = ay;
        if (heading) {
            if (psi_in) po = g_psi[t];  // state.psi (:310)
            const double raw = atan2_fast(s, c);
            const double two_pi = 6.283185307179586;
            // np.round((psi - raw) / 2 pi): the quotient is within 1 ulp of the reference's (exactly
            // representable halves never occur in practice), multiply by the rounded reciprocal
            const double tgt = raw + two_pi * rint((po - raw) * 0.15915494309189535);
            T[kTgt * n_p] = tgt;
            if (MODE == kModeHeading && A.s.psi_targets) A.s.psi_targets[i * n_p + t] = tgt;
        }
    }
    __syncthreads();

    // ---------------- heading QP (:311-314)
    if (heading) {
        constexpr int kHs = 8;
        const int chunk = (n_p + kHs - 1) / kHs;
        for (int w = tid; w < m * kHs; w += kB2Threads) {
            const int k = w % m, q = w / m;
            const int t1 = min(n_p, (q + 1) * chunk);
            double acc = 0.0;
            for (int t = q * chunk; t < t1; ++t) acc = fma(__ldg(Pr + t * m + k), sT[kTgt * n_p + t], acc);
            sPart[q * m + k] = acc;
        }
        __syncthreads();
        if (tid < m) {
            double acc = 0.0;
            for (int q = 0; q < kHs; ++q) acc += sPart[q * m + tid];
            sRp[tid] = -(-g_lp[tid] - rho_p * acc);
        } else if (tid < m + 2) {
            sRp[tid] = A.c.b_psi[tid - m];
        }
        __syncthreads();
        if (tid < m) {
            const double* K = A.c.kinvT_psi + (int64_t)level * (m + 2) * m + tid;
            double acc = 0.0;
            for (int j = 0; j < m + 2; ++j) acc = fma(__ldg(K + j * m), sRp[j], acc);
            sPn[tid] = acc;
            if (MODE == kModeHeading) g_xp[tid] = acc;
        }
        __syncthreads();
        if (MODE == kModeHeading) {
            if (g_psi)
                for (int t = tid; t < n_p; t += kB2Threads) {
                    double psi = 0.0;
#pragma unroll kB2UnrollM
                    for (int k = 0; k < kB2MaxM; ++k) {
                        if (k >= m) break;
                        psi = fma(__ldg(PT + k * n_p + t), sPn[k], psi);
                    }
                    g_psi[t] = psi;
                }
            return;
        }
    }
    if (!body) return;

    // ---------------- body: per sample, rows of F xi - g
    double rmax = 0.0, ss = 0.0;
    double dmin = __longlong_as_double(0x7ff0000000000000LL), vmax2 = 0.0, amax2 = 0.0, cost_s = 0.0, cost_t = 0.0;
    const double vmx = A.c.v_max, amx = A.c.a_max;
    for (int t = tid; t < n_p; t += kB2Threads) {
        double* T = sT + t;
        const double x = T[kX * n_p], y = T[kY * n_p], c = T[kC * n_p], s = T[kS * n_p];
        const double vx = T[kVX * n_p], vy = T[kVY * n_p], ax = T[kAX * n_p], ay = T[kAY * n_p];
        double psi = 0.0, pacc = 0.0;
        if (!iter && psi_in) {
            psi = g_psi[t];
        } else {
#pragma unroll kB2UnrollM
            for (int k = 0; k < kB2MaxM; ++k) {
                if (k >= m) break;
                psi = fma(__ldg(PT + k * n_p + t), sPn[k], psi);
            }
        }
        if (MODE == kModeRank)
            for (int k = 0; k < m; ++k) pacc = fma(__ldg(PddT + k * n_p + t), sPn[k], pacc);
        double sp, cp;
        sincos_fast(psi, &sp, &cp);
        const int64_t o1 = i * n_p + t;
        // velocity / acceleration rows: alpha = atan2 (unit vector), d clipped to [0, 1] (:325-344)
        double cav, sav, caa, saa;
        if (given_alpha) {
            sincos_fast(A.s.alpha_v[o1], &sav, &cav);
            sincos_fast(A.s.alpha_a[o1], &saa, &caa);
        } else {
            unit2(vx, vy, &cav, &sav);
            unit2(ax, ay, &caa, &saa);
        }
        double dv, da;
        if (given_d) {
            dv = A.s.d_v[o1];
            da = A.s.d_a[o1];
        } else {
            dv = clip((vx * cav + vy * sav) / vmx, 0.0, 1.0);
            da = clip((ax * caa + ay * saa) / amx, 0.0, 1.0);
        }
        const double gvx = vmx * dv * cav, gvy = vmx * dv * sav;
        const double gax = amx * da * caa, gay = amx * da * saa;
        const double rvx = vx - gvx, rvy = vy - gvy, rax = ax - gax, ray = ay - gay;
        // heading copy rows [0, P] xi_c = cos(psi) (:225-226)
        const double rhx = c - cp, rhy = s - sp;
        rmax = dmax(dmax(dmax(rmax, fabs(rvx)), fabs(rvy)), dmax(fabs(rax), fabs(ray)));
        rmax = dmax(rmax, dmax(fabs(rhx), fabs(rhy)));
        ss = fma(rvx, rvx, ss);
        ss = fma(rvy, rvy, ss);
        ss = fma(rax, rax, ss);
        ss = fma(ray, ray, ss);
        ss = fma(rhx, rhx, ss);
        ss = fma(rhy, rhy, ss);
        if (MODE == kModeMaterialise) {
            if (!given_alpha) {
                if (A.s.alpha_v) A.s.alpha_v[o1] = atan2_fast(vy, vx);
                if (A.s.alpha_a) A.s.alpha_a[o1] = atan2_fast(ay, ax);
            }
            if (A.s.d_v) A.s.d_v[o1] = dv;
            if (A.s.d_a) A.s.d_a[o1] = da;
        }
        if ((MODE == kModeMaterialise || MODE == kModeRank) && !psi_in && g_psi) g_psi[t] = psi;
        // collision rows, per circle then obstacle
        double Gx = 0, Gy = 0, Gcx = 0, Gcy = 0, Rx = 0, Ry = 0, Rcx = 0, Rcy = 0;
        for (int ci = 0; ci < n_c; ++ci) {
            const double r = __ldg(A.c.offsets + ci);
            const double cx = fma(r, cp, x), cy = fma(r, sp, y);  // circle centre (:200-201)
            const double fx = fma(r, c, x), fy = fma(r, s, y);    // F row [P, r P] xi (:155)
            double gxs = 0, gys = 0, rxs = 0, rys = 0;
            if (CIRC) {
                // Circles (a == b): the clamp d >= 1 is inactive iff h >= a, and then the target is the
                // circle centre itself, g = o + a (h / a) (dx, dy) / h = c (:221-222, :338-340), so only the
                // clamped (inside) elements need the closed forms; the rest contribute k * c to the sums
                // and the obstacle-independent residual (fx - cx, fy - cy).
                int k_out = 0;
                const double* op = A.c.obs + t;
                auto element = [&](int o, double ox, double oy) {
                    const double dx = cx - ox, dy = cy - oy;
                    const double h2 = fma(dx, dx, dy * dy);
                    const double2 lim = reinterpret_cast<const double2*>(sAI)[o];  // (a^2, (1e6 a)^2)
                    if (h2 >= lim.x && h2 <= lim.y) {
                        ++k_out;
                        return;
                    }
                    const double a = sAB[5 * o];
                    double ex, ey;
                    if (h2 > 0.0) {
                        const double rr = rsqrt_fast(h2);
                        const double sc = a * clip(h2 * rr * sAB[5 * o + 4], 1.0, 1.0e6) * rr;
                        ex = dx * sc;
                        ey = dy * sc;
                    } else {  // atan2(+-0, +-0) conventions (unit2), d = 1
                        ex = flip_sign(a, sign_bit(dx));
                        ey = flip_sign(0.0, sign_bit(dy));
                    }
                    const double gx = ox + ex, gy = oy + ey;
                    const double rx = fx - gx, ry = fy - gy;
                    gxs += gx;
                    gys += gy;
                    rxs += rx;
                    rys += ry;
                    rmax = dmax(dmax(rmax, fabs(rx)), fabs(ry));
                    ss = fma(rx, rx, ss);
                    ss = fma(ry, ry, ss);
                };
                constexpr int kBatch = B2_OBS_BATCH;  // all loads of a batch in flight before the first use
                const int stride = 2 * n_p;
                int o = 0;
                for (; o + kBatch <= n_o; o += kBatch) {
                    double ox[kBatch], oy[kBatch];
#pragma unroll
                    for (int j = 0; j < kBatch; ++j) {
                        ox[j] = __ldg(op + (o + j) * stride);
                        oy[j] = __ldg(op + (o + j) * stride + n_p);
                    }
#pragma unroll
                    for (int j = 0; j < kBatch; ++j) element(o + j, ox[j], oy[j]);
                }
                for (; o < n_o; ++o) element(o, __ldg(op + o * stride), __ldg(op + o * stride + n_p));
                if (k_out) {
                    const double kd = (double)k_out, rx = fx - cx, ry = fy - cy;
                    gxs = fma(kd, cx, gxs);
                    gys = fma(kd, cy, gys);
                    rxs = fma(kd, rx, rxs);
                    rys = fma(kd, ry, rys);
                    rmax = dmax(dmax(rmax, fabs(rx)), fabs(ry));
                    ss = fma(kd, fma(rx, rx, ry * ry), ss);
                }
            } else {
            const double* op = A.c.obs + t;
            const double* const op_last = op + (int64_t)(n_o > 0 ? n_o - 1 : 0) * 2 * n_p;
            double ox_n = n_o > 0 ? __ldg(op) : 0.0, oy_n = n_o > 0 ? __ldg(op + n_p) : 0.0;
            for (int o = 0; o < n_o; ++o) {
                const double ox = ox_n, oy = oy_n;  // prefetched one obstacle ahead
                op = op < op_last ? op + 2 * n_p : op;
                ox_n = __ldg(op);
                oy_n = __ldg(op + n_p);
                const double dx = cx - ox, dy = cy - oy;
                double ex, ey, d;
                {
                    const double* ab = sAB + 5 * o;
                    const int64_t oe = ((i * n_c + ci) * n_o + o) * n_p + t;
                    if (given_alpha) {
                        double ca, sa;
                        sincos_fast(A.s.alpha_coll[oe], &sa, &ca);
                        if (given_d) {
                            d = A.s.d_coll[oe];
                        } else {
                            const double num = ab[0] * dx * ca + ab[1] * dy * sa;
                            const double den = ab[2] * (ca * ca) + ab[3] * (sa * sa);
                            d = clip(num / den, 1.0, 1.0e6);  // :338-340
                        }
                        ex = ab[0] * d * ca;
                        ey = ab[1] * d * sa;
                    } else {
                        b2_element(dx, dy, ab, ab[0] == ab[1], &ex, &ey, &d);
                    }
                    if (MODE == kModeMaterialise) {
                        if (!given_alpha && A.s.alpha_coll) A.s.alpha_coll[oe] = atan2_fast(dy, dx);
                        if (A.s.d_coll) A.s.d_coll[oe] = d;
                    }
                    if (MODE == kModeRank) dmin = fmin(dmin, hypot(dx / ab[0], dy / ab[1]));  // :387-388
                }
                const double gx = ox + ex, gy = oy + ey;  // :221-222
                const double rx = fx - gx, ry = fy - gy;
                gxs += gx;
                gys += gy;
                rxs += rx;
                rys += ry;
                rmax = dmax(dmax(rmax, fabs(rx)), fabs(ry));
                ss = fma(rx, rx, ss);
                ss = fma(ry, ry, ss);
            }
            }
            Gx += gxs;
            Gy += gys;
            Gcx = fma(r, gxs, Gcx);
            Gcy = fma(r, gys, Gcy);
            Rx += rxs;
            Ry += rys;
            Rcx = fma(r, rxs, Rcx);
            Rcy = fma(r, rys, Rcy);
        }
        if (MODE == kModeRank) {
            vmax2 = fmax(vmax2, hypot(vx, vy));
            amax2 = fmax(amax2, hypot(ax, ay));
            cost_s += ax * ax + ay * ay + pacc * pacc;
            const double ex = x - __ldg(A.c.desired + 2 * t), ey = y - __ldg(A.c.desired + 2 * t + 1);
            cost_t += ex * ex + ey * ey;
        }
        if (MODE <= kModePrime) {
            T[kGVX * n_p] = gvx;
            T[kGVY * n_p] = gvy;
            T[kGAX * n_p] = gax;
            T[kGAY * n_p] = gay;
            T[kGX * n_p] = Gx;
            T[kGY * n_p] = Gy;
            T[kGCX * n_p] = Gcx + cp;
            T[kGCY * n_p] = Gcy + sp;
        }
        if (iter) {
            T[kRVX * n_p] = rvx;
            T[kRVY * n_p] = rvy;
            T[kRAX * n_p] = rax;
            T[kRAY * n_p] = ray;
            T[kRX * n_p] = Rx;
            T[kRY * n_p] = Ry;
            T[kRCX * n_p] = Rcx + rhx;
            T[kRCY * n_p] = Rcy + rhy;
            T[kDPsi * n_p] = psi - T[kTgt * n_p];
            if (g_psi) g_psi[t] = psi;
        }
    }
    if (MODE == kModeMaterialise) return;

    // ---------------- per-member residual max / norm
    rmax = warp_max(rmax);
    ss = warp_sum(ss);
    if (MODE == kModeRank) {
        for (int o = 16; o > 0; o >>= 1) {
            dmin = fmin(dmin, __shfl_xor_sync(0xffffffffu, dmin, o));
            vmax2 = fmax(vmax2, __shfl_xor_sync(0xffffffffu, vmax2, o));
            amax2 = fmax(amax2, __shfl_xor_sync(0xffffffffu, amax2, o));
        }
        cost_s = warp_sum(cost_s);
        cost_t = warp_sum(cost_t);
    }
    __shared__ double s_rank[kB2Warps][5];
    if (lane == 0) {
        sRed[warp] = rmax;
        sRed[kB2Warps + warp] = ss;
        if (MODE == kModeRank) {
            s_rank[warp][0] = dmin;
            s_rank[warp][1] = vmax2;
            s_rank[warp][2] = amax2;
            s_rank[warp][3] = cost_s;
            s_rank[warp][4] = cost_t;
        }
    }
    __syncthreads();
    if (MODE == kModeRank) {
        if (tid == 0) {
            double mm = sRed[0], s2 = sRed[kB2Warps], dm = s_rank[0][0], v2 = s_rank[0][1], a2 = s_rank[0][2];
            double cs = s_rank[0][3], ct = s_rank[0][4];
            for (int w = 1; w < kB2Warps; ++w) {
                mm = fmax(mm, sRed[w]);
                s2 += sRed[kB2Warps + w];
                dm = fmin(dm, s_rank[w][0]);
                v2 = fmax(v2, s_rank[w][1]);
                a2 = fmax(a2, s_rank[w][2]);
                cs += s_rank[w][3];
                ct += s_rank[w][4];
            }
            double* rk = A.s.rank + i * 6;
            rk[0] = mm;
            rk[1] = sqrt(s2);
            rk[2] = dm;
            rk[3] = v2;
            rk[4] = a2;
            rk[5] = A.c.w_smooth * cs + A.c.w_track * ct;  // _member_costs (:366-374)
        }
        return;
    }

    // ---------------- contractions: F'g (iterate, prime), F'r and P'(psi - targets) (iterate)
    // contraction: out[k][col] = sum_t M[t][k] T[col][t] for M = P (9 columns), Pdot (4), Pddot (4);
    // thread (k, q) keeps all columns of one basis row k over t-chunk q in registers (one basis
    // load per sample feeds every column), partials summed over q in a fixed order.
    {
        constexpr int kQ = kB2Q;
        const int chunk = (n_p + kQ - 1) / kQ;
        const int ncol = iter ? 17 : 8;
        for (int w = tid; w < m * kQ; w += kB2Threads) {
            const int k = w % m, q = w / m;
            const int t0 = q * chunk, t1 = min(n_p, t0 + chunk);
            double aP[9], aD[4], aA[4];
#pragma unroll
            for (int c = 0; c < 9; ++c) aP[c] = 0.0;
#pragma unroll
            for (int c = 0; c < 4; ++c) aD[c] = 0.0, aA[c] = 0.0;
            for (int t = t0; t < t1; ++t) {
                const double p = __ldg(Pr + t * m + k), pd = __ldg(Pdr + t * m + k), pdd = __ldg(Pddr + t * m + k);
                const double* T = sT + t;
                aD[0] = fma(pd, T[kGVX * n_p], aD[0]);
                aD[1] = fma(pd, T[kGVY * n_p], aD[1]);
                aA[0] = fma(pdd, T[kGAX * n_p], aA[0]);
                aA[1] = fma(pdd, T[kGAY * n_p], aA[1]);
                aP[0] = fma(p, T[kGX * n_p], aP[0]);
                aP[1] = fma(p, T[kGY * n_p], aP[1]);
                aP[2] = fma(p, T[kGCX * n_p], aP[2]);
                aP[3] = fma(p, T[kGCY * n_p], aP[3]);
                if (iter) {
                    aD[2] = fma(pd, T[kRVX * n_p], aD[2]);
                    aD[3] = fma(pd, T[kRVY * n_p], aD[3]);
                    aA[2] = fma(pdd, T[kRAX * n_p], aA[2]);
                    aA[3] = fma(pdd, T[kRAY * n_p], aA[3]);
                    aP[4] = fma(p, T[kRX * n_p], aP[4]);
                    aP[5] = fma(p, T[kRY * n_p], aP[5]);
                    aP[6] = fma(p, T[kRCX * n_p], aP[6]);
                    aP[7] = fma(p, T[kRCY * n_p], aP[7]);
                    aP[8] = fma(p, T[kDPsi * n_p], aP[8]);
                }
            }
            // outputs: [g: x c y s | r: x c y s | psi], each block m wide
            double* out = sPart + q * (2 * nv + m);
            out[k] = (aD[0] + aA[0]) + aP[0];
            out[m + k] = aP[2];
            out[2 * m + k] = (aD[1] + aA[1]) + aP[1];
            out[3 * m + k] = aP[3];
            if (iter) {
                out[nv + k] = (aD[2] + aA[2]) + aP[4];
                out[nv + m + k] = aP[6];
                out[nv + 2 * m + k] = (aD[3] + aA[3]) + aP[5];
                out[nv + 3 * m + k] = aP[7];
                out[2 * nv + k] = aP[8];
            }
            (void)ncol;
        }
        __syncthreads();
        const int n_out = iter ? 2 * nv + m : nv;
        for (int u = tid; u < n_out; u += kB2Threads) {
            double acc = 0.0;
            for (int q = 0; q < kQ; ++q) acc += sPart[q * (2 * nv + m) + u];
            sOut[u] = acc;
        }
        __syncthreads();
    }
    if (tid < nv) {
        g_sum[tid] = sOut[tid];
        if (iter) {
            g_xi[tid] = sXi[tid];
            g_lam[tid] = g_lam[tid] - rho * sOut[nv + tid];  // :359
        }
    }
    if (iter && tid < m) {
        g_xp[tid] = sPn[tid];
        g_lp[tid] = g_lp[tid] - rho_p * sOut[2 * nv + tid];  // :360-361
    }
    if (tid == 0) {
        double mm = sRed[0], s2 = sRed[kB2Warps];
        for (int w = 1; w < kB2Warps; ++w) {
            mm = fmax(mm, sRed[w]);
            s2 += sRed[kB2Warps + w];
        }
        A.s.res_max[i] = mm;
        A.s.res_norm[i] = sqrt(s2);
    }
    if (!iter) return;

    // ---------------- last CTA: batch-global bookkeeping (:451-461), one warp
    if (warp != 0) return;
    unsigned last = 0;
    if (lane == 0) {
        __threadfence();
        last = atomicAdd(A.s.counter, 1u) == (unsigned)(A.d.n_members - 1);
    }
    last = __shfl_sync(0xffffffffu, last, 0);
    if (!last) return;
    __threadfence();
    b2_batch_epilogue(A, level, rho);
    if (lane == 0) *A.s.counter = 0u;
}

template <int NC, int MODE, bool CIRC = false>
static int b2_launch(const B2Args& A, size_t smem, cudaStream_t st) {
    static bool attr_set[64] = {false};
    int dev = 0;
    cudaGetDevice(&dev);
    if (smem > 48 * 1024 && dev >= 0 && dev < 64 && !attr_set[dev]) {
        cudaFuncSetAttribute(b2_kernel<NC, MODE, CIRC>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
        attr_set[dev] = true;
    }
    b2_kernel<NC, MODE, CIRC><<<(unsigned)A.d.n_members, kB2Threads, smem, st>>>(A);
    return (int)cudaGetLastError();
}

template <int NC>
static int b2_dispatch(const B2Args& A, int mode, size_t smem, cudaStream_t st) {
    // the circle path only for the implied-geometry modes (given alpha / d need the general one)
    const bool circ = (A.p.flags & TRO_B2_CIRCLES) && !(A.p.flags & (TRO_B2_GIVEN_AD | TRO_B2_GIVEN_ALPHA));
    switch (mode) {
        case kModeIter:
            return circ ? b2_launch<NC, kModeIter, true>(A, smem, st) : b2_launch<NC, kModeIter>(A, smem, st);
        case kModePrime:
            return circ ? b2_launch<NC, kModePrime, true>(A, smem, st) : b2_launch<NC, kModePrime>(A, smem, st);
        case kModeMaterialise: return b2_launch<NC, kModeMaterialise>(A, smem, st);
        case kModeRank: return b2_launch<NC, kModeRank>(A, smem, st);
        case kModeXi: return b2_launch<NC, kModeXi>(A, smem, st);
        default: return b2_launch<NC, kModeHeading>(A, smem, st);
    }
}

}  // namespace tro

extern "C" int tro_b2_run(int32_t mode, const tro_b2_dims* d, const tro_b2_consts* c, const tro_b2_state* s,
                          const tro_b2_params* p, void* stream) {
    if (!d || !c || !s || !p || mode < 0 || mode > 6) return TRO_EINVAL;
    if (!c->k_xi || !c->kinvT_xi) return TRO_EINVAL;  // the xi step solves with K^-1 and refines with K
    if ((p->flags & TRO_B2_SHARD) && mode == 0 && !s->shard) return TRO_EINVAL;
    if (mode == 6) {
        if (!s->shards_in || p->n_shards < 1 || !s->ring || p->stall_window < 1 ||
            2 * p->stall_window > tro::kB2MaxRing)
            return TRO_EINVAL;
        tro::B2Args A1;
        A1.d = *d;
        A1.c = *c;
        A1.s = *s;
        A1.p = *p;
        tro::b2_merge_kernel<<<1, 32, 0, reinterpret_cast<cudaStream_t>(stream)>>>(A1);
        return (int)cudaGetLastError();
    }
    if (d->n_c < 1 || d->n_c > tro::kB2MaxC || d->n_obs < 0 || d->n_p < 2 || d->m < 1 || d->n_levels < 1)
        return TRO_EINVAL;
    if (d->m > tro::kB2MaxM) return TRO_EINVAL;
    if (mode == 0 && (p->stall_window < 1 || 2 * p->stall_window > tro::kB2MaxRing || !s->counter || !s->ring))
        return TRO_EINVAL;
    if (mode == 3 && !s->rank) return TRO_EINVAL;
    if ((p->flags & TRO_B2_PSI_IN) && !s->psi) return TRO_EINVAL;
    if ((mode == 1 || mode == 3) && (p->flags & TRO_B2_GIVEN_AD) &&
        (!s->alpha_coll || !s->d_coll || !s->alpha_v || !s->alpha_a || !s->d_v || !s->d_a))
        return TRO_EINVAL;
    if (mode == 2 && (p->flags & TRO_B2_GIVEN_ALPHA) && (!s->alpha_coll || !s->alpha_v || !s->alpha_a))
        return TRO_EINVAL;
    if (d->n_members <= 0) return 0;
    if (d->n_members > 0x7fffffffLL) return TRO_EINVAL;
    tro::B2Args A;
    A.d = *d;
    A.c = *c;
    A.s = *s;
    A.p = *p;
    const tro::B2Smem L = tro::b2_layout(d->n_p, d->m, d->n_obs);
    const size_t smem = (size_t)L.total * sizeof(double);
    if (smem > 200 * 1024) return TRO_EINVAL;
    cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
    if (d->n_c == 1) return tro::b2_dispatch<1>(A, mode, smem, st);
    return tro::b2_dispatch<0>(A, mode, smem, st);
}
