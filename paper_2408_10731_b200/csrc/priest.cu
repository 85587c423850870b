// PRIEST projection-guided sampling + CEM baseline (arXiv 2408.10731, Alg. 3) for sm_100a.
//
// The projection (solver_priest.py:242-287) is FP-pipe bound, not HBM bound:
// a sample's whole problem (33 coefficients, its 100x100 obstacle/sample grid
// of polar targets, 30 inner iterations) stays on chip.  One warp owns one
// sample for all inner iterations; a CTA of 8 warps shares the basis, K^-1,
// F'F and the obstacle shapes in shared memory.  Per inner iteration a warp:
//   1. evaluates pos/vel/acc of its xi at every sample t (lanes own t),
//   2. walks the obstacles: polar target in trig-free form
//        e = c + (d/q) (p - c),  q = ellipsoidal norm of p - c,  d = clip(q, 1, 1e6)
//      (== obs + a d cos(alpha) sin(beta), ... of solver_priest.py:202-210; for
//      q >= 1 the target is the position itself), accumulating sum_j e and the
//      residual score,
//   3. the velocity/acceleration targets v min(1, v_max/|v|) and the box slack,
//   4. F'e (warp butterflies), lambda -= rho (F'F xi - F'e),
//      q_lin = -(samples + lambda + rho F'e), xi = K^-1 [-q_lin; b_eq].
// The last obstacle remainder of n_p (100 = 3*32 + 4) is split over obstacle
// groups so all 32 lanes stay busy.
#include "common.cuh"
#include "fastmath.cuh"
#include "../../include/trajopt_b200.h"

namespace tro {

#ifndef PR_WARPS
#define PR_WARPS 8
#endif
constexpr int kPrWarps = PR_WARPS;  // samples (warps) per CTA
#ifndef PR_KB
#define PR_KB 4  // obstacles per batch of scaled distances (C4: 2 / 3 / 4 / 6 / 8 -> 7.37 / 6.66 / 6.53 / 6.64 / 7.00 ms)
#endif
#ifndef PR_MINB
#define PR_MINB 2  // 2 CTAs / SM at the 128-register cap (3 spills heavily)
#endif
constexpr int kPrMaxDm = 48;  // dim * m
constexpr int kPrMaxNk = 72;  // dim * m + n_eq

struct PrArgs {
    tro_priest_dims d;
    tro_priest_consts c;
    tro_priest_io io;
};

struct PrSmem {
    int P, Pd, Pdd, kinv, M, obs, wbuf, vec, total;  // doubles
};
// obstacles: 8 doubles each: cx cy cz 1/a^2 1/b^2 a b -   (centres only meaningful for static tracks)
__host__ __device__ inline PrSmem pr_layout(int n_p, int m, int dim, int nk, int n_o, bool wbuf) {
    PrSmem L;
    int off = 0;
    L.P = off;    off += n_p * m;
    L.Pd = off;   off += n_p * m;
    L.Pdd = off;  off += n_p * m;
    L.kinv = off; off += dim * m * nk;                 // only the xi rows of K^-1
    L.M = off;    off += m * m;
    off = (off + 1) & ~1;  // 16-byte aligned obstacle records (double2 loads)
    L.obs = off;  off += 8 * (n_o > 0 ? n_o : 1);
    L.wbuf = off; off += wbuf ? kPrWarps * 3 * dim * n_p : 0;  // runtime-m path: F' weights per (blk, ax, t)
    L.vec = off;  off += kPrWarps * 5 * kPrMaxNk;     // per warp: xi, lam, samp, fte, rhs
    L.total = off;
    return L;
}

__device__ __forceinline__ double warp_allsum(double v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    return v;
}

// Polar target of an obstacle the point is INSIDE of (or absurdly far from):
// e = c + (d/q) (p - c), d = clip(q, 1, 1e6); q == 0 -> the pole (atan2(0, 0) = 0,
// solver_priest.py:204-210).  Accumulates e into S and |p - e|^2 into r2.
template <int DIM>
__device__ __forceinline__ void inside_target(const double* p, const double* dl, const double* c, double q2,
                                              double a, double b, double* S, double& r2) {
    double e[3];
    if (q2 == 0.0) {
#pragma unroll
        for (int k = 0; k < DIM; ++k) e[k] = c[k];
        if constexpr (DIM == 3) e[2] = c[2] + b;
        else e[0] = c[0] + a;
    } else {
        const double rs = rsqrt_fast(q2);
        const double f = q2 < 1.0 ? rs : 1e6 * rs;
#pragma unroll
        for (int k = 0; k < DIM; ++k) e[k] = fma(f, dl[k], c[k]);
    }
#pragma unroll
    for (int k = 0; k < DIM; ++k) {
        S[k] += e[k];
        const double r = p[k] - e[k];
        r2 = fma(r, r, r2);
    }
}

// velocity / acceleration polar target limit * clip(|v|/limit, 0, 1) * v/|v| (solver_priest.py:219-235)
template <int DIM>
__device__ __forceinline__ void speed_target(const double* v, double limit, double* e, double& r2) {
    double s2 = 0.0;
#pragma unroll
    for (int k = 0; k < DIM; ++k) s2 = fma(v[k], v[k], s2);
    if (s2 <= limit * limit) {
#pragma unroll
        for (int k = 0; k < DIM; ++k) e[k] = v[k];
        return;
    }
    const double f = limit * rsqrt_fast(s2);
#pragma unroll
    for (int k = 0; k < DIM; ++k) {
        e[k] = f * v[k];
        const double r = v[k] - e[k];
        r2 = fma(r, r, r2);
    }
}

// M: compile-time basis columns (0 = runtime m, F'e via a shared-memory weight buffer);
// STATIC: obstacle centres constant over the horizon (kept in shared memory).
template <int DIM, int M, bool STATIC, bool SPH>
__global__ void __launch_bounds__(kPrWarps * 32, PR_MINB) priest_project_kernel(PrArgs A) {
    extern __shared__ double smem[];
    const int n_p = A.d.n_p, n_o = A.d.n_obs, neq = A.d.n_eq;
    const int m = M ? M : A.d.m;
    const int dm = DIM * m, nk = dm + neq;
    const PrSmem L = pr_layout(n_p, m, DIM, nk, n_o, M == 0);
    double* sP = smem + L.P;
    double* sPd = smem + L.Pd;
    double* sPdd = smem + L.Pdd;
    double* sK = smem + L.kinv;
    double* sM = smem + L.M;
    double* sObs = smem + L.obs;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;

    for (int k = tid; k < n_p * m; k += blockDim.x) {
        sP[k] = ld_const(A.c.P + k);
        sPd[k] = ld_const(A.c.Pd + k);
        sPdd[k] = ld_const(A.c.Pdd + k);
    }
    for (int k = tid; k < dm * nk; k += blockDim.x) sK[k] = ld_const(A.c.kinv + k);
    for (int k = tid; k < m * m; k += blockDim.x) sM[k] = ld_const(A.c.FtF + k);
    for (int k = tid; k < n_o; k += blockDim.x) {
        const double a = ld_const(A.c.shape_a + k), b = ld_const(A.c.shape_b + k);
        double* o = sObs + 8 * k;
        for (int q = 0; q < 3; ++q) o[q] = (STATIC && q < DIM) ? ld_const(A.c.tracks + ((int64_t)k * DIM + q) * n_p) : 0.0;
        o[3] = 1.0 / (a * a);
        o[4] = 1.0 / (b * b);
        o[5] = a;
        o[6] = b;
    }
    __syncthreads();

    const int64_t s = (int64_t)blockIdx.x * kPrWarps + warp;  // this warp's sample
    if (s >= A.d.n_samples) return;
    double* xi = smem + L.vec + warp * 5 * kPrMaxNk;
    double* lam = xi + kPrMaxNk;
    double* smp = lam + kPrMaxNk;
    double* fte = smp + kPrMaxNk;
    double* rhs = fte + kPrMaxNk;
    double* W = smem + L.wbuf + warp * 3 * DIM * n_p;  // M == 0 only

    // ---- the sample: samples = mu + z L' (numpy multivariate_normal(svd)), or given
    for (int c = lane; c < dm; c += 32) {
        double v;
        if (A.io.z) {
            const double* zr = A.io.z + s * dm;
            v = 0.0;
            for (int q = 0; q < dm; ++q) v = fma(zr[q], ld_const(A.c.draw_L + c * dm + q), v);
            v += A.c.mu[c];
        } else {
            v = A.io.samples[s * dm + c];
        }
        smp[c] = v;
        xi[c] = v;
        lam[c] = 0.0;
        if (A.io.samples_out) A.io.samples_out[s * dm + c] = v;
    }
    __syncwarp();
    if (A.d.n_inner < 0) {  // draw only (the CEM baseline samples without projecting)
        for (int c = lane; c < dm; c += 32) A.io.xi[s * dm + c] = smp[c];
        return;
    }

    const bool has_v = A.c.v_max > 0.0, has_a = A.c.a_max > 0.0, has_b = A.c.has_bounds != 0;
    const int full_slots = n_p / 32;
    const int rem = n_p - 32 * full_slots;
    const int ng = (rem > 0 && (32 % rem) == 0) ? 32 / rem : 1;  // obstacle groups of the remainder slot
    const int nslots = full_slots + (rem ? 1 : 0);
    const double rho = A.c.rho;
    const int n_inner = A.d.n_inner;
    constexpr int DMC = M ? DIM * M : 1;

    for (int it = 0; it <= n_inner; ++it) {
        // ---------- targets of the current xi: F'e contributions and the residual score
        double r2 = 0.0;
        double facc[DMC];
#pragma unroll
        for (int c = 0; c < DMC; ++c) facc[c] = 0.0;
        for (int u = 0; u < nslots; ++u) {
            const bool remslot = (u == full_slots);
            int t, jg = 0, jstep = 1;
            bool active = true;
            if (!remslot) {
                t = 32 * u + lane;
            } else if (ng > 1) {
                t = 32 * u + lane % rem;
                jg = lane / rem;
                jstep = ng;
            } else {
                t = 32 * u + lane;
                active = lane < rem;
            }
            if (!active) t = 0;  // keep the (discarded) reads in bounds
            double p[3] = {0, 0, 0}, v[3] = {0, 0, 0}, ac[3] = {0, 0, 0};
#pragma unroll
            for (int k = 0; k < DIM; ++k) {
                double ps = 0.0, vs = 0.0, as = 0.0;
                for (int c = 0; c < m; ++c) {
                    const double x = xi[k * m + c];
                    ps = fma(sP[t * m + c], x, ps);
                    vs = fma(sPd[t * m + c], x, vs);
                    as = fma(sPdd[t * m + c], x, as);
                }
                p[k] = ps;
                v[k] = vs;
                ac[k] = as;
            }
            double S[3] = {0, 0, 0};
            double rr = 0.0;
            int outside = 0;
            if (active) {
                const double* tr = A.c.tracks + t;
                // the scaled distances of kB obstacles first (independent: ILP across obstacles), then the
                // rare inside targets; ncu showed the one-obstacle-at-a-time chain stalled on fixed latency
                constexpr int kB = PR_KB;
                auto q2_of = [&](int j, double* dl, double* cc) -> double {
                    const double* o = sObs + 8 * j;
                    double ia2;
                    if constexpr (STATIC) {
                        const double2 c01 = reinterpret_cast<const double2*>(o)[0];
                        const double2 c2i = reinterpret_cast<const double2*>(o)[1];
                        cc[0] = c01.x;
                        cc[1] = c01.y;
                        cc[2] = c2i.x;
                        ia2 = c2i.y;
                    } else {
#pragma unroll
                        for (int k = 0; k < DIM; ++k) cc[k] = ld_const(tr + ((int64_t)j * DIM + k) * n_p);
                        ia2 = o[3];
                    }
#pragma unroll
                    for (int k = 0; k < DIM; ++k) dl[k] = p[k] - cc[k];
                    if constexpr (SPH) {  // a == b: one multiplier, no 1/b^2 load
                        if constexpr (DIM == 3) return fma(dl[2], dl[2], fma(dl[1], dl[1], dl[0] * dl[0])) * ia2;
                        else return fma(dl[1], dl[1], dl[0] * dl[0]) * ia2;
                    }
                    if constexpr (DIM == 3) return fma(dl[2] * dl[2], o[4], (dl[0] * dl[0] + dl[1] * dl[1]) * ia2);
                    else return fma(dl[1] * dl[1], o[4], dl[0] * dl[0] * ia2);
                };
                int j = jg;
                for (; j + (kB - 1) * jstep < n_o; j += kB * jstep) {
                    double q2[kB];
#pragma unroll
                    for (int u = 0; u < kB; ++u) {
                        double dl[3], cc[3];
                        q2[u] = q2_of(j + u * jstep, dl, cc);
                    }
                    // outside (target == the point itself, added once below): branch-free count; the rare
                    // inside elements are handled behind one branch per batch
                    unsigned inside = 0;
#pragma unroll
                    for (int u = 0; u < kB; ++u) {
                        // 1 <= q2 < 2^40 (the high word below 1e12's) as one 32-bit unsigned range test on the
                        // bit pattern (q2 >= 0, so the patterns are monotone; NaN and 0 fall outside): integer
                        // pipe, two instructions; the sliver [hi(1e12), 1e12] is settled exactly below
                        const unsigned hi = (unsigned)__double2hiint(q2[u]);
                        inside |= (hi - 0x3FF00000u < 0x426D1A94u - 0x3FF00000u) ? 0u : (1u << u);
                    }
                    outside += kB - __popc(inside);
                    if (inside) {  // per-lane (lanes of the remainder slot walk different obstacle groups)
#pragma unroll
                        for (int u = 0; u < kB; ++u) {
                            if (inside & (1u << u)) {  // recompute the offsets (keeping kB live costs registers)
                                double dl[3], cc[3];
                                const double qq = q2_of(j + u * jstep, dl, cc);
                                if (qq >= 1.0 && qq <= 1e12) {  // the exact test (reached only near 1e12)
                                    ++outside;
                                } else {
                                    const double* o = sObs + 8 * (j + u * jstep);
                                    inside_target<DIM>(p, dl, cc, qq, o[5], o[6], S, rr);
                                }
                            }
                        }
                    }
                }
                for (; j < n_o; j += jstep) {
                    double dl[3], cc[3];
                    const double q2 = q2_of(j, dl, cc);
                    if (q2 >= 1.0 && q2 <= 1e12) {
                        ++outside;
                    } else {
                        const double* o = sObs + 8 * j;
                        inside_target<DIM>(p, dl, cc, q2, o[5], o[6], S, rr);
                    }
                }
#pragma unroll
                for (int k = 0; k < DIM; ++k) S[k] = fma((double)outside, p[k], S[k]);
            }
            if (remslot && ng > 1) {  // combine the obstacle groups of the remainder slot
                for (int o = rem; o < 32; o <<= 1) {
#pragma unroll
                    for (int k = 0; k < DIM; ++k) S[k] += __shfl_xor_sync(0xffffffffu, S[k], o);
                }
                active = jg == 0;  // one writer per t; the score partials stay per lane
            }
            r2 += rr;
            double w0[3] = {0, 0, 0}, w1[3] = {0, 0, 0}, w2[3] = {0, 0, 0};
            if (active) {
                if (has_v) speed_target<DIM>(v, A.c.v_max, w1, r2);
                if (has_a) speed_target<DIM>(ac, A.c.a_max, w2, r2);
#pragma unroll
                for (int k = 0; k < DIM; ++k) {
                    double wp = S[k];
                    if (has_b) {
                        // box rows G = [-P; P], tau = [-s_min; s_max] (solver_priest.py:142-150, 265-268)
                        const double lo = A.c.s_min[k], hi = A.c.s_max[k];
                        const double e_lo = -lo - fmax(0.0, p[k] - lo);
                        const double e_hi = hi - fmax(0.0, hi - p[k]);
                        wp += e_hi - e_lo;
                        const double vl = fmax(0.0, lo - p[k]), vh = fmax(0.0, p[k] - hi);
                        r2 = fma(vl, vl, fma(vh, vh, r2));
                    }
                    w0[k] = wp;
                }
            }
            if constexpr (M > 0) {
                if (active) {
#pragma unroll
                    for (int c = 0; c < M; ++c) {
                        const double pp = sP[t * M + c], pd = sPd[t * M + c], pa = sPdd[t * M + c];
#pragma unroll
                        for (int k = 0; k < DIM; ++k)
                            facc[k * M + c] = fma(pa, w2[k], fma(pd, w1[k], fma(pp, w0[k], facc[k * M + c])));
                    }
                }
            } else if (active) {
#pragma unroll
                for (int k = 0; k < DIM; ++k) {
                    W[(0 * DIM + k) * n_p + t] = w0[k];
                    W[(1 * DIM + k) * n_p + t] = w1[k];
                    W[(2 * DIM + k) * n_p + t] = w2[k];
                }
            }
        }
        r2 = warp_allsum(r2);
        if (it > 0 && A.io.history && lane == 0) A.io.history[(int64_t)(it - 1) * A.d.n_samples + s] = sqrt(r2);
        if (it == n_inner) {
            if (lane == 0) A.io.scores[s] = sqrt(r2);
            break;
        }

        // ---------- F'e : per coefficient, the sum over t of the weighted basis rows
        if constexpr (M > 0) {
#pragma unroll
            for (int c = 0; c < DMC; ++c) facc[c] = warp_allsum(facc[c]);
            if (lane == 0) {
#pragma unroll
                for (int c = 0; c < DMC; ++c) fte[c] = facc[c];
            }
        } else {
            __syncwarp();
            for (int c = 0; c < dm; ++c) {
                const int k = c / m, cc = c - k * m;
                double acc = 0.0;
                for (int t = lane; t < n_p; t += 32) {
                    acc = fma(sP[t * m + cc], W[(0 * DIM + k) * n_p + t], acc);
                    acc = fma(sPd[t * m + cc], W[(1 * DIM + k) * n_p + t], acc);
                    acc = fma(sPdd[t * m + cc], W[(2 * DIM + k) * n_p + t], acc);
                }
                acc = warp_allsum(acc);
                if (lane == 0) fte[c] = acc;
            }
        }
        __syncwarp();
        // ---------- lambda -= rho F'(F xi - e);  rhs = [-q_lin ; b_eq] (solver_priest.py:271-274)
        for (int c = lane; c < dm; c += 32) {
            const int k = c / m, cc = c - k * m;
            double ftfx = 0.0;
            for (int q = 0; q < m; ++q) ftfx = fma(sM[cc * m + q], xi[k * m + q], ftfx);
            const double l = lam[c] - rho * (ftfx - fte[c]);
            lam[c] = l;
            rhs[c] = smp[c] + l + rho * fte[c];  // = -q_lin
        }
        for (int e = lane; e < neq; e += 32) rhs[dm + e] = A.c.b_eq[e];
        __syncwarp();
        for (int c = lane; c < dm; c += 32) {
            double acc = 0.0;
            for (int q = 0; q < nk; ++q) acc = fma(sK[c * nk + q], rhs[q], acc);
            xi[c] = acc;
        }
        __syncwarp();
    }
    for (int c = lane; c < dm; c += 32) A.io.xi[s * dm + c] = xi[c];
}

// ---------------------------------------------------------------- batched costs
// barn_cost (solver_priest.py:475-498) of selected samples (+ residual weight * score)
// and the CEM penalty (solver_priest.py:396-419).  One warp per sample.
template <int DIM>
__global__ void __launch_bounds__(256) priest_cost_kernel(PrArgs A, const double* __restrict__ xis,
                                                          const int64_t* __restrict__ index, int64_t count,
                                                          const double* __restrict__ scores, double w_barn,
                                                          double w_score, double w_penalty, double* __restrict__ out) {
    const int lane = threadIdx.x & 31;
    const int64_t r = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    if (r >= count) return;
    const int n_p = A.d.n_p, m = A.d.m, n_o = A.d.n_obs;
    const int dm = DIM * m;
    const int64_t s = index ? index[r] : r;
    const double* xi = xis + s * dm;
    const double* ls = A.c.line;  // start xy, end xy
    const double ax_ = ls[2] - ls[0], ay_ = ls[3] - ls[1];
    const double len = sqrt(ax_ * ax_ + ay_ * ay_);
    const double ux = len < 1e-12 ? 0.0 : ax_ / len, uy = len < 1e-12 ? 0.0 : ay_ / len;
    double smooth = 0.0, ck = 0.0, cp = 0.0, pen = 0.0;
    for (int t = lane; t < n_p; t += 32) {
        double p[3] = {0, 0, 0}, v[3] = {0, 0, 0}, ac[3] = {0, 0, 0};
        for (int k = 0; k < DIM; ++k) {
            for (int c = 0; c < m; ++c) {
                const double x = xi[k * m + c];
                p[k] = fma(ld_const(A.c.P + t * m + c), x, p[k]);
                v[k] = fma(ld_const(A.c.Pd + t * m + c), x, v[k]);
                ac[k] = fma(ld_const(A.c.Pdd + t * m + c), x, ac[k]);
            }
        }
        if (w_barn != 0.0) {  // barn cost terms (xy only)
            smooth += ac[0] * ac[0] + ac[1] * ac[1];
            const double sp = hypot(v[0], v[1]);
            if (sp > 1e-6) {
                const double kap = (ac[1] * v[0] - ac[0] * v[1]) / (sp * sp * sp);
                ck += kap * kap;
            }
            const double rx = p[0] - ls[0], ry = p[1] - ls[1];
            double d2 = rx * rx + ry * ry;
            if (len >= 1e-12) {
                const double al = rx * ux + ry * uy;
                d2 -= al * al;
            }
            cp += fmax(d2, 0.0);
        }
        if (w_penalty != 0.0) {
            const double* tr = A.c.tracks + t;
            for (int j = 0; j < n_o; ++j) {
                const double a = ld_const(A.c.shape_a + j), b = ld_const(A.c.shape_b + j);
                double qd = 0.0;
                for (int k = 0; k < DIM; ++k) {
                    const double dl = p[k] - ld_const(tr + ((int64_t)j * DIM + k) * n_p);
                    qd += dl * dl / ((k < 2 && DIM == 3) || k == 0 ? a * a : b * b);
                }
                pen += fmax(0.0, 1.0 - qd);
            }
            if (A.c.v_max > 0.0) pen += fmax(0.0, v[0] * v[0] + v[1] * v[1] + (DIM == 3 ? v[2] * v[2] : 0.0) -
                                                      A.c.v_max * A.c.v_max);
            if (A.c.a_max > 0.0) pen += fmax(0.0, ac[0] * ac[0] + ac[1] * ac[1] + (DIM == 3 ? ac[2] * ac[2] : 0.0) -
                                                      A.c.a_max * A.c.a_max);
            if (A.c.has_bounds)
                for (int k = 0; k < DIM; ++k)
                    pen += fmax(0.0, A.c.s_min[k] - p[k]) + fmax(0.0, p[k] - A.c.s_max[k]);
        }
    }
    smooth = warp_allsum(smooth);
    ck = warp_allsum(ck);
    cp = warp_allsum(cp);
    pen = warp_allsum(pen);
    if (lane == 0) {
        double c = w_barn != 0.0 ? w_barn * (smooth + ck + cp) : 0.0;
        if (scores) c += w_score * scores[s];
        out[r] = c + w_penalty * pen;
    }
}

// ---------------------------------------------------------------- distribution refit
// weights = exp((c - min c)/gamma); mu' = (1-sigma) mu + sigma sum(w x)/sum w;
// Sigma' = (1-sigma) Sigma + sigma sum(w (x - mu')(x - mu')')/sum w   (solver_priest.py:317-333)
// cem = true selects the plain CEM refit (mean, population covariance; :442-444); otherwise gamma is used as
// given (gamma == 0 gives numpy's exp(x / 0): inf / NaN weights), and min(c) propagates NaN like np.min.
__global__ void __launch_bounds__(256) elite_update_kernel(const double* __restrict__ xis, int dm,
                                                           const int64_t* __restrict__ rows, int n_el,
                                                           const double* __restrict__ costs, double sigma,
                                                           double gamma, int cem, double* mu, double* cov) {
    __shared__ double w[1024];
    __shared__ double mnew[kPrMaxDm];
    __shared__ double red[2];
    const int tid = threadIdx.x;
    if (tid == 0) {
        double cmin = costs[0];
        for (int k = 1; k < n_el; ++k) {
            const double c = costs[k];
            if (cmin == cmin && (c != c || c < cmin)) cmin = c;  // np.min: NaN wins
        }
        double ws = 0.0;
        for (int k = 0; k < n_el; ++k) {
            const double v = !cem ? exp((costs[k] - cmin) / gamma) : 1.0;
            w[k] = v;
            ws += v;
        }
        red[0] = ws;
    }
    __syncthreads();
    const double ws = red[0];
    for (int c = tid; c < dm; c += blockDim.x) {
        double acc = 0.0;
        for (int k = 0; k < n_el; ++k) acc += w[k] * xis[rows[k] * dm + c];
        const double wm = acc / ws;
        const double nm = !cem ? (1.0 - sigma) * mu[c] + sigma * wm : wm;
        mnew[c] = nm;
    }
    __syncthreads();
    for (int o = tid; o < dm * dm; o += blockDim.x) {
        const int a = o / dm, b = o - a * dm;
        double acc = 0.0;
        for (int k = 0; k < n_el; ++k) {
            const double* x = xis + rows[k] * dm;
            acc += w[k] * ((x[a] - mnew[a]) * (x[b] - mnew[b]));
        }
        const double wc = acc / ws;
        cov[o] = !cem ? (1.0 - sigma) * cov[o] + sigma * wc : wc;
    }
    __syncthreads();
    for (int c = tid; c < dm; c += blockDim.x) mu[c] = mnew[c];
}

// ---------------------------------------------------------------- throughput-mode sampling
// Philox4x32-10 (Salmon et al., SC'11: the counter-based generator of cuRAND / numpy's Philox) keyed by
// the 64-bit seed; counter = (pair index (64 bit), stream id (64 bit)).  Each counter gives two 53-bit
// uniforms and, by Box-Muller, two standard normals, so element e of sample s is a pure function of
// (seed, stream, s * ceil(d / 2) * 2 + j): any shard of the batch draws its own samples.
__device__ __forceinline__ void philox10(uint32_t c[4], uint32_t k0, uint32_t k1) {
#pragma unroll
    for (int r = 0; r < 10; ++r) {
        const uint32_t h0 = __umulhi(0xD2511F53u, c[0]), l0 = 0xD2511F53u * c[0];
        const uint32_t h1 = __umulhi(0xCD9E8D57u, c[2]), l1 = 0xCD9E8D57u * c[2];
        const uint32_t n0 = h1 ^ c[1] ^ k0, n2 = h0 ^ c[3] ^ k1;
        c[0] = n0;
        c[1] = l1;
        c[2] = n2;
        c[3] = l0;
        k0 += 0x9E3779B9u;
        k1 += 0xBB67AE85u;
    }
}

__global__ void normal_philox_kernel(uint64_t seed, uint64_t stream_id, int64_t first, int64_t n, int d,
                                     double* __restrict__ out) {
    const int dp = (d + 1) / 2;  // counters per sample
    const int64_t total = n * dp;
    for (int64_t q = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; q < total; q += (int64_t)gridDim.x * blockDim.x) {
        const int64_t s = q / dp;
        const int h = (int)(q - s * dp);
        const uint64_t ctr = (uint64_t)(first + s) * dp + h;
        uint32_t c[4] = {(uint32_t)ctr, (uint32_t)(ctr >> 32), (uint32_t)stream_id, (uint32_t)(stream_id >> 32)};
        philox10(c, (uint32_t)seed, (uint32_t)(seed >> 32));
        // uniforms in (0, 1]: 53 bits each
        const uint64_t a = ((uint64_t)c[0] << 21) ^ (c[1] >> 11), b = ((uint64_t)c[2] << 21) ^ (c[3] >> 11);
        const double u1 = ((double)(a & ((1ull << 53) - 1)) + 1.0) * 0x1.0p-53;
        const double u2 = (double)(b & ((1ull << 53) - 1)) * 0x1.0p-53;
        const double r = sqrt(-2.0 * log(u1));
        double sn, cs;
        sincospi(2.0 * u2, &sn, &cs);
        double* o = out + s * d + 2 * h;
        o[0] = r * cs;
        if (2 * h + 1 < d) o[1] = r * sn;
    }
}

// Cholesky factor L (lower, row-major) of a symmetric positive semidefinite n x n matrix, one CTA: columns
// left to right; a pivot <= 0 (a singular direction of the refit covariance) gives a zero column, so
// L L' == A on the matrix's range.  Throughput-mode draw factor (samples = mu + z L'), in place of numpy's
// svd factor u sqrt(s) (same distribution, not the same samples).
__global__ void __launch_bounds__(256) cholesky_kernel(const double* __restrict__ A, int n, double* __restrict__ L) {
    __shared__ double s[kPrMaxDm * kPrMaxDm];
    for (int k = threadIdx.x; k < n * n; k += blockDim.x) s[k] = A[k];
    __syncthreads();
    for (int j = 0; j < n; ++j) {
        __shared__ double piv;
        if (threadIdx.x == 0) {
            const double v = s[j * n + j];
            piv = v > 0.0 ? sqrt(v) : 0.0;
            s[j * n + j] = piv;
        }
        __syncthreads();
        for (int i = j + 1 + threadIdx.x; i < n; i += blockDim.x) s[i * n + j] = piv > 0.0 ? s[i * n + j] / piv : 0.0;
        __syncthreads();
        for (int o = threadIdx.x; o < (n - j - 1) * (n - j - 1); o += blockDim.x) {
            const int i = j + 1 + o / (n - j - 1), k = j + 1 + o % (n - j - 1);
            if (k <= i) s[i * n + k] -= s[i * n + j] * s[k * n + j];
        }
        __syncthreads();
    }
    for (int k = threadIdx.x; k < n * n; k += blockDim.x) {
        const int i = k / n, c = k - i * n;
        L[k] = c <= i ? s[k] : 0.0;
    }
}

}  // namespace tro

// ---------------------------------------------------------------- C-ABI
static int pr_check(const tro_priest_dims* d) {
    if (!d || (d->dim != 2 && d->dim != 3) || d->m < 1 || d->n_p < 2 || d->n_obs < 0 || d->n_samples < 0 ||
        d->n_inner < -1)
        return TRO_EINVAL;
    if (d->dim * d->m > tro::kPrMaxDm || d->dim * d->m + d->n_eq > tro::kPrMaxNk) return TRO_EINVAL;
    return 0;
}

template <int DIM, int M, bool STATIC>
static void pr_launch(const tro::PrArgs& A, unsigned blocks, size_t smem, cudaStream_t st) {
    if (A.c.spheres) {
        cudaFuncSetAttribute(tro::priest_project_kernel<DIM, M, STATIC, true>,
                             cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        tro::priest_project_kernel<DIM, M, STATIC, true><<<blocks, tro::kPrWarps * 32, smem, st>>>(A);
        return;
    }
    cudaFuncSetAttribute(tro::priest_project_kernel<DIM, M, STATIC, false>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         (int)smem);
    tro::priest_project_kernel<DIM, M, STATIC, false><<<blocks, tro::kPrWarps * 32, smem, st>>>(A);
}

template <int DIM>
static void pr_dispatch(const tro::PrArgs& A, unsigned blocks, size_t smem, cudaStream_t st) {
    const bool stat = A.c.static_tracks != 0;
    switch (A.d.m) {
        case 11: stat ? pr_launch<DIM, 11, true>(A, blocks, smem, st) : pr_launch<DIM, 11, false>(A, blocks, smem, st); break;
        case 9: stat ? pr_launch<DIM, 9, true>(A, blocks, smem, st) : pr_launch<DIM, 9, false>(A, blocks, smem, st); break;
        default: stat ? pr_launch<DIM, 0, true>(A, blocks, smem, st) : pr_launch<DIM, 0, false>(A, blocks, smem, st);
    }
}

extern "C" int tro_priest_project_f64(const tro_priest_dims* dims, const tro_priest_consts* c, const tro_priest_io* io,
                                      void* stream) {
    if (pr_check(dims) || !c || !io || !io->xi || !io->scores || (!io->z && !io->samples)) return TRO_EINVAL;
    if (dims->n_samples == 0) return 0;
    tro::PrArgs A;
    A.d = *dims;
    A.c = *c;
    A.io = *io;
    const int nk = dims->dim * dims->m + dims->n_eq;
    const bool wbuf = !(dims->m == 9 || dims->m == 11);
    const tro::PrSmem L = tro::pr_layout(dims->n_p, dims->m, dims->dim, nk, dims->n_obs, wbuf);
    const size_t smem = (size_t)L.total * sizeof(double);
    if (smem > 227 * 1024) return TRO_EINVAL;
    const unsigned blocks = (unsigned)((dims->n_samples + tro::kPrWarps - 1) / tro::kPrWarps);
    cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
    if (dims->dim == 3) pr_dispatch<3>(A, blocks, smem, st);
    else pr_dispatch<2>(A, blocks, smem, st);
    return (int)cudaGetLastError();
}

extern "C" int tro_priest_cost_f64(const tro_priest_dims* dims, const tro_priest_consts* c, const double* xis,
                                   const int64_t* index, int64_t count, const double* scores, double w_barn,
                                   double w_score, double w_penalty, double* out, void* stream) {
    if (pr_check(dims) || !c || !xis || !out || count < 0) return TRO_EINVAL;
    if (count == 0) return 0;
    tro::PrArgs A;
    A.d = *dims;
    A.c = *c;
    const unsigned blocks = (unsigned)((count * 32 + 255) / 256);
    cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
    if (dims->dim == 3)
        tro::priest_cost_kernel<3><<<blocks, 256, 0, st>>>(A, xis, index, count, scores, w_barn, w_score, w_penalty,
                                                            out);
    else
        tro::priest_cost_kernel<2><<<blocks, 256, 0, st>>>(A, xis, index, count, scores, w_barn, w_score, w_penalty,
                                                            out);
    return (int)cudaGetLastError();
}

extern "C" int tro_elite_update_f64(const double* xis, int32_t dm, const int64_t* rows, int32_t n_elite,
                                    const double* costs, double sigma, double gamma, int32_t mode, double* mu,
                                    double* cov, void* stream) {
    if (!xis || !rows || !costs || !mu || !cov || dm < 1 || dm > tro::kPrMaxDm || n_elite < 1 || n_elite > 1024 ||
        (mode != TRO_REFIT_PRIEST && mode != TRO_REFIT_CEM))
        return TRO_EINVAL;
    tro::elite_update_kernel<<<1, 256, 0, reinterpret_cast<cudaStream_t>(stream)>>>(
        xis, dm, rows, n_elite, costs, sigma, gamma, mode == TRO_REFIT_CEM, mu, cov);
    return (int)cudaGetLastError();
}

extern "C" int tro_normal_philox_f64(uint64_t seed, uint64_t stream_id, int64_t first_sample, int64_t n_samples,
                                     int32_t dim, double* out, void* stream) {
    if (!out || n_samples < 0 || first_sample < 0 || dim < 1) return TRO_EINVAL;
    if (n_samples == 0) return 0;
    const int64_t total = n_samples * ((dim + 1) / 2);
    int64_t blocks = (total + 255) / 256;
    if (blocks > 148 * 8) blocks = 148 * 8;
    tro::normal_philox_kernel<<<(unsigned)blocks, 256, 0, reinterpret_cast<cudaStream_t>(stream)>>>(
        seed, stream_id, first_sample, n_samples, dim, out);
    return (int)cudaGetLastError();
}

extern "C" int tro_cholesky_f64(const double* a, int32_t n, double* l, void* stream) {
    if (!a || !l || n < 1 || n > tro::kPrMaxDm) return TRO_EINVAL;
    tro::cholesky_kernel<<<1, 256, 0, reinterpret_cast<cudaStream_t>(stream)>>>(a, n, l);
    return (int)cudaGetLastError();
}
