// Shared device helpers for libtrajopt_b200 (sm_100a).
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

namespace tro {

// ---- math overloads: the per-element arithmetic runs in the storage type T
__device__ __forceinline__ void sincos_t(double x, double* s, double* c) { sincos(x, s, c); }
__device__ __forceinline__ void sincos_t(float x, float* s, float* c) { sincosf(x, s, c); }
__device__ __forceinline__ double atan2_t(double y, double x) { return atan2(y, x); }
__device__ __forceinline__ float atan2_t(float y, float x) { return atan2f(y, x); }
__device__ __forceinline__ double sqrt_t(double x) { return sqrt(x); }
__device__ __forceinline__ float sqrt_t(float x) { return sqrtf(x); }
__device__ __forceinline__ double fmin_t(double a, double b) { return fmin(a, b); }
__device__ __forceinline__ float fmin_t(float a, float b) { return fminf(a, b); }
__device__ __forceinline__ double fmax_t(double a, double b) { return fmax(a, b); }
__device__ __forceinline__ float fmax_t(float a, float b) { return fmaxf(a, b); }
__device__ __forceinline__ double fabs_t(double a) { return fabs(a); }
__device__ __forceinline__ float fabs_t(float a) { return fabsf(a); }

// ---- streaming global access (state is touched once per iteration and is
// larger than L2 at the benchmark sizes: evict-first)
__device__ __forceinline__ double ld_stream(const double* p) { return __ldcs(p); }
__device__ __forceinline__ float ld_stream(const float* p) { return __ldcs(p); }
__device__ __forceinline__ void st_stream(double* p, double v) { __stcs(p, v); }
__device__ __forceinline__ void st_stream(float* p, float v) { __stcs(p, v); }

// read-only constants (tracks, basis, K^-1): keep in L2
__device__ __forceinline__ double ld_const(const double* p) { return __ldg(p); }

__device__ __forceinline__ double warp_sum(double v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    return v;
}
__device__ __forceinline__ double warp_max(double v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v = fmax(v, __shfl_xor_sync(0xffffffffu, v, o));
    return v;
}

// np.mean of the w ring values v[k] = ring[(start + k) % w2], k = 0 .. w-1, with numpy's own summation
// order (pairwise_sum in numpy/_core/src/umath/loops_utils.h.src, which np.add.reduce uses for float64):
// n < 8 sequential from 0.0; 8 <= n <= 128 eight interleaved partial sums combined as
// ((r0 + r1) + (r2 + r3)) + ((r4 + r5) + (r6 + r7)), then the n % 8 tail in order; then / n.
// (The stall windows here are <= 32, so the recursive n > 128 branch never applies.)
__device__ __forceinline__ double np_mean_ring(const double* ring, int start, int w, int w2) {
    // ring index of window element k: (start + k) mod w2, one division for the whole window
    int i0 = start % w2;
    auto at = [&](int k) {
        int idx = i0 + k;
        if (idx >= w2) idx -= w2;
        return ring[idx];
    };
    double res;
    if (w < 8) {
        res = 0.0;
        for (int k = 0; k < w; ++k) res += at(k);
    } else {
        double r[8];
#pragma unroll
        for (int j = 0; j < 8; ++j) r[j] = at(j);
        int k = 8;
        for (; k < w - (w % 8); k += 8) {
#pragma unroll
            for (int j = 0; j < 8; ++j) r[j] += at(k + j);
        }
        res = ((r[0] + r[1]) + (r[2] + r[3])) + ((r[4] + r[5]) + (r[6] + r[7]));
        for (; k < w; ++k) res += at(k);
    }
    return res / (double)w;
}

}  // namespace tro
