// Batched post-solve validation for sm_100a.
//
// The reference evaluates each trajectory in Python against the RAW scenario geometry
// (bench/metrics.py:26-95): smoothness sum(acc^2), tracking sum((pos - desired)^2), arc length
// sum |pos[t+1] - pos[t]|, the worst incursion max(1 + margin - dist) and the clearance lower bound
// min((dist - 1) min(a, b)) with dist the ellipsoidal distance sqrt(dx^2/a^2 + dy^2/a^2 [+ dz^2/b^2])
// to every obstacle's constant-velocity track (scenarios.py:118-127).  Here one warp owns one member:
// positions / accelerations come from the coefficients (P xi, Pddot xi as 8x8x4 fp64 tensor-core tiles, the
// member's coefficients held as the B fragments) or from given samples; the (sample, obstacle) distance
// pass keeps up to 4 of a lane's samples in registers per broadcast obstacle record and spreads the < 32
// tail samples over the lanes by obstacle; obstacle centres are predicted on the fly (c + v (t - t0)).
// Every sum runs in a fixed order and the rest are exact minima, so a member's numbers do not depend on
// the batch.
#include <type_traits>

#include "common.cuh"
#include "fastmath.cuh"
#include "../../include/trajopt_b200.h"

namespace tro {

#ifndef VAL_WARPS
#define VAL_WARPS 8  // members per CTA: 2 -> 51 M, 4 -> 60 M, 8 -> 61.5 M, 16 -> 60 M traj/s (val config)
#endif
constexpr int kValWarps = VAL_WARPS;  // members per CTA (fewer when the sample buffers would not fit)
constexpr int kValRec = 9;     // doubles per obstacle record

// D(8x8) += A(8x4, row) B(4x8, col), fp64 tensor cores (lane l: A[l/4][l%4], B[l%4][l/4], D[l/4][2 (l%4) + j])
__device__ __forceinline__ void dmma884_v(double* d, double a, double b) {
    asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0, %1}, {%2}, {%3}, {%0, %1};"
                 : "+d"(d[0]), "+d"(d[1])
                 : "d"(a), "d"(b));
}

struct ValArgs {
    tro_val_dims d;
    tro_val_consts c;
    tro_val_io io;
};

template <int DIM>
__global__ void __launch_bounds__(kValWarps * 32) validate_kernel(ValArgs A) {
    extern __shared__ double smem[];
    const int n_p = A.d.n_p, m = A.d.m, n_o = A.d.n_obs;
    const bool coeffs = A.io.xi != nullptr;
    double* sP = smem;                         // n_p x m   (coefficient mode)
    double* sPdd = sP + n_p * m;               // n_p x m
    double* sObs = sPdd + n_p * m;             // n_o x 8: c(3) v(3) inv a^2... see below
    double* sPos = sObs + kValRec * (n_o > 0 ? n_o : 1);  // kValWarps x n_p x DIM
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    if (coeffs)
        for (int k = tid; k < n_p * m; k += blockDim.x) {
            sP[k] = __ldg(A.c.P + k);
            sPdd[k] = __ldg(A.c.Pdd + k);
        }
    // obstacle record: centre (3), velocity (3), 1/a^2, 1/b^2, min(a, b)
    for (int j = tid; j < n_o; j += blockDim.x) {
        double* o = sObs + kValRec * j;
        for (int k = 0; k < 3; ++k) {
            o[k] = k < DIM ? __ldg(A.c.centers + j * DIM + k) : 0.0;
            o[3 + k] = k < DIM ? __ldg(A.c.velocities + j * DIM + k) : 0.0;
        }
        const double a = __ldg(A.c.shape_a + j), b = __ldg(A.c.shape_b + j);
        o[6] = 1.0 / (a * a);
        o[7] = 1.0 / (b * b);
        o[8] = a < b ? a : b;
    }
    __syncthreads();
    // one clearance scale min(a, b) for every obstacle (the common case): then worst and the clearance
    // bound are monotone functions of the smallest scaled square distance, so one sqrt per member suffices
    __shared__ int s_uniform;
    if (tid == 0) {
        int u = 1;
        for (int j = 1; j < n_o; ++j) u &= sObs[kValRec * j + 8] == sObs[8];
        s_uniform = u;
    }
    __syncthreads();
    const bool uniform = s_uniform != 0;
    const int64_t i = (int64_t)blockIdx.x * (blockDim.x >> 5) + warp;  // one member per warp
    if (i >= A.d.n_members) return;
    double* pw = sPos + (int64_t)warp * n_p * DIM;
    const double* xi = coeffs ? A.io.xi + i * DIM * m : nullptr;
    const double t0_time = __ldg(A.c.t);
    double smooth = 0.0, track = 0.0;
    double qmin = __longlong_as_double(0x7ff0000000000000LL), clear = qmin;
    if (coeffs) {
        // positions and accelerations on the fp64 tensor cores: [P | Pdd](t, c) x xi(c, axis) as 8x8x4 tiles
        // (t = tile row, axis = tile column); the member's coefficients are the B fragments, loaded once
        const int ksn = (m + 3) >> 2;  // m <= 16 (tro_validate_f64)
        double bx[4];
#pragma unroll
        for (int ks = 0; ks < 4; ++ks) {
            const int c = 4 * ks + (lane & 3), ax = lane >> 2;
            bx[ks] = (ks < ksn && c < m && ax < DIM) ? __ldg(xi + ax * m + c) : 0.0;
        }
        for (int mt = 0; mt < (n_p + 7) >> 3; ++mt) {
            double dp[2] = {0.0, 0.0}, da[2] = {0.0, 0.0};
            const int ta = mt * 8 + (lane >> 2);
#pragma unroll
            for (int ks = 0; ks < 4; ++ks) {
                if (ks < ksn) {
                    const int c = 4 * ks + (lane & 3);
                    const bool ok = ta < n_p && c < m;
                    dmma884_v(dp, ok ? sP[ta * m + c] : 0.0, bx[ks]);
                    dmma884_v(da, ok ? sPdd[ta * m + c] : 0.0, bx[ks]);
                }
            }
            const int td = mt * 8 + (lane >> 2), ax0 = 2 * (lane & 3);
#pragma unroll
            for (int j = 0; j < 2; ++j) {
                if (td < n_p && ax0 + j < DIM) {
                    pw[td * DIM + ax0 + j] = dp[j];
                    smooth = fma(da[j], da[j], smooth);
                }
            }
        }
    } else {
        for (int t = lane; t < n_p; t += 32) {
#pragma unroll
            for (int k = 0; k < DIM; ++k) {
                pw[t * DIM + k] = __ldg(A.io.pos + (i * n_p + t) * DIM + k);
                const double ac = __ldg(A.io.acc + (i * n_p + t) * DIM + k);
                smooth = fma(ac, ac, smooth);
            }
        }
    }
    __syncwarp();
    if (A.c.desired)
        for (int t = lane; t < n_p; t += 32) {
            const double* dd = A.c.desired + (A.d.per_member_desired ? (i * n_p + t) * DIM : (int64_t)t * DIM);
#pragma unroll
            for (int k = 0; k < DIM; ++k) {
                const double e = pw[t * DIM + k] - __ldg(dd + k);
                track = fma(e, e, track);
            }
        }
    // obstacle distances: every (sample, obstacle) pair, all reductions are minima (exact, order-free), so lanes
    // can take any partition.  Full groups of 32 samples: each lane keeps up to 4 of its samples in registers
    // and reuses one broadcast obstacle record for all of them; the < 32 tail samples are spread over the
    // lanes by obstacle instead (no idle lanes at n_p = 100).
    const double* tt = A.c.t;
    auto element = [&](const double* o, double p0, double p1, double p2, double tau) {
        double q = 0.0;
#pragma unroll
        for (int k = 0; k < DIM; ++k) {
            const double d = (k == 0 ? p0 : k == 1 ? p1 : p2) - fma(o[3 + k], tau, o[k]);
            // metrics.py:63-65: the last axis uses b (z in 3-D, y in 2-D), the others a; multiplied by the
            // reciprocal squares (<= 1 ulp per term from the reference's divisions)
            q = fma(d * d, k == DIM - 1 ? o[7] : o[6], q);
        }
        qmin = q < qmin ? q : qmin;
        if (!uniform) {
            const double cl = (sqrt(q) - 1.0) * o[8];
            clear = cl < clear ? cl : clear;
        }
    };
    auto group = [&](auto ns_tag, int t0) {
        constexpr int NS = decltype(ns_tag)::value;
        double pp[NS][3], tau[NS];
#pragma unroll
        for (int u = 0; u < NS; ++u) {
            const int t = t0 + 32 * u + lane;
#pragma unroll
            for (int k = 0; k < 3; ++k) pp[u][k] = k < DIM ? pw[t * DIM + k] : 0.0;
            tau[u] = __ldg(tt + t) - t0_time;  // predict_obstacles: c + v (t_now + t - t0), t_now = 0
        }
        for (int j = 0; j < n_o; ++j) {
            const double* o = sObs + kValRec * j;
#pragma unroll
            for (int u = 0; u < NS; ++u) element(o, pp[u][0], pp[u][1], pp[u][2], tau[u]);
        }
    };
    const int n_full = n_p >> 5;
    int g = 0;
    for (; g + 4 <= n_full; g += 4) group(std::integral_constant<int, 4>{}, 32 * g);
    switch (n_full - g) {
        case 3: group(std::integral_constant<int, 3>{}, 32 * g); break;
        case 2: group(std::integral_constant<int, 2>{}, 32 * g); break;
        case 1: group(std::integral_constant<int, 1>{}, 32 * g); break;
        default: break;
    }
    for (int t = 32 * n_full; t < n_p; ++t) {  // tail samples: lanes over obstacles
        const double* pp = pw + t * DIM;
        double pt[3];
#pragma unroll
        for (int k = 0; k < 3; ++k) pt[k] = k < DIM ? pp[k] : 0.0;
        const double tau = __ldg(tt + t) - t0_time;
        for (int j = lane; j < n_o; j += 32) element(sObs + kValRec * j, pt[0], pt[1], pt[2], tau);
    }
    __syncwarp();
    // arc length over the warp's stored positions (metrics.py:39-40), fixed order: lanes own segments
    double arc = 0.0;
    for (int t = lane; t + 1 < n_p; t += 32) {
        double s = 0.0;
#pragma unroll
        for (int k = 0; k < DIM; ++k) {
            const double e = pw[(t + 1) * DIM + k] - pw[t * DIM + k];
            s = fma(e, e, s);
        }
        arc += sqrt(s);
    }
    smooth = warp_sum(smooth);
    track = warp_sum(track);
    arc = warp_sum(arc);
    for (int o = 16; o > 0; o >>= 1) {
        const double oq = __shfl_xor_sync(0xffffffffu, qmin, o), oc = __shfl_xor_sync(0xffffffffu, clear, o);
        qmin = oq < qmin ? oq : qmin;
        clear = oc < clear ? oc : clear;
    }
    // max(1 + margin - dist) = 1 + margin - sqrt(min q) (sqrt and the affine maps are monotone, also rounded)
    const double dmin = sqrt(qmin);
    const double worst = n_o > 0 ? (1.0 + A.c.margin) - dmin : -__longlong_as_double(0x7ff0000000000000LL);
    if (uniform && n_o > 0) clear = (dmin - 1.0) * sObs[8];
    if (lane == 0) {
        double* out = A.io.out + i * 5;
        out[0] = smooth;
        out[1] = track;
        out[2] = arc;
        out[3] = worst;   // -inf without obstacles (check_collision_free)
        out[4] = clear;   // +inf without obstacles (clearance_lower_bound)
    }
}

}  // namespace tro

extern "C" int tro_validate_f64(const tro_val_dims* d, const tro_val_consts* c, const tro_val_io* io, void* stream) {
    if (!d || !c || !io || !io->out || (d->dim != 2 && d->dim != 3) || d->n_p < 2 || d->n_obs < 0 || !c->t)
        return TRO_EINVAL;
    if (io->xi ? (d->m < 1 || d->m > 16 || !c->P || !c->Pdd) : (!io->pos || !io->acc)) return TRO_EINVAL;
    if (d->n_obs > 0 && (!c->centers || !c->velocities || !c->shape_a || !c->shape_b)) return TRO_EINVAL;
    if (d->n_members <= 0) return 0;
    tro::ValArgs A;
    A.d = *d;
    A.c = *c;
    A.io = *io;
    const int m = io->xi ? d->m : 0;
    // members (warps) per CTA: kValWarps, halved while the per-warp sample buffers do not fit
    int wpc = tro::kValWarps;
    auto smem_for = [&](int w) {
        return sizeof(double) * ((size_t)2 * d->n_p * m + tro::kValRec * (d->n_obs > 0 ? d->n_obs : 1) +
                                 (size_t)w * d->n_p * d->dim);
    };
    while (wpc > 1 && smem_for(wpc) > 200 * 1024) wpc >>= 1;
    const size_t smem = smem_for(wpc);
    if (smem > 200 * 1024) return TRO_EINVAL;
    const unsigned blocks = (unsigned)((d->n_members + wpc - 1) / wpc);
    if (d->dim == 3)
        cudaFuncSetAttribute(tro::validate_kernel<3>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    else
        cudaFuncSetAttribute(tro::validate_kernel<2>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
    if (d->dim == 3)
        tro::validate_kernel<3><<<blocks, wpc * 32, smem, st>>>(A);
    else
        tro::validate_kernel<2><<<blocks, wpc * 32, smem, st>>>(A);
    return (int)cudaGetLastError();
}
