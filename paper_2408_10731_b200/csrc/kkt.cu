// Batched KKT-inverse application: the drop-in for qpcore.solve_batch
// (qpcore.py:130-143).  out[c] = K^-1 rhs[c] for every right-hand side c, where
// rhs[c] = [-q_c ; b_c] and K^-1 is the explicit fp64 inverse of the saddle
// matrix (computed once per factorization by the host from the same LU).
//
// fp64 throughout (TF32 loses 0.35 relative on these
// ill-conditioned saddles).  A CTA stages K^-1 (n <= 64) and a tile of 64
// right-hand sides in shared memory; each thread produces outputs with the
// row of K^-1 broadcast from shared memory.
#include "common.cuh"
#include "../../include/trajopt_b200.h"

namespace tro {

constexpr int kTileCols = 64;
constexpr int kSmemMaxN = 64;

__global__ void __launch_bounds__(256) kkt_apply_small(const double* __restrict__ kinv, int n,
                                                         const double* __restrict__ rhs, int64_t ncols,
                                                         double* __restrict__ out) {
    extern __shared__ double sm[];
    double* sK = sm;              // n x n
    double* sR = sm + n * n;      // kTileCols x (n + 1) (padded against bank conflicts)
    const int ld = n + 1;
    const int64_t c0 = (int64_t)blockIdx.x * kTileCols;
    const int cols = (ncols - c0) < kTileCols ? (int)(ncols - c0) : kTileCols;
    for (int k = threadIdx.x; k < n * n; k += blockDim.x) sK[k] = __ldg(kinv + k);
    for (int k = threadIdx.x; k < cols * n; k += blockDim.x) {
        const int c = k / n, r = k - c * n;
        sR[c * ld + r] = rhs[(c0 + c) * n + r];
    }
    __syncthreads();
    for (int k = threadIdx.x; k < cols * n; k += blockDim.x) {
        const int c = k / n, r = k - c * n;
        const double* Kr = sK + r * n;
        const double* x = sR + c * ld;
        double acc = 0.0;
        for (int q = 0; q < n; ++q) acc += Kr[q] * x[q];
        out[(c0 + c) * n + r] = acc;
    }
}

// generic n: one warp per (column, row-chunk); K^-1 rows streamed from L2
__global__ void __launch_bounds__(256) kkt_apply_large(const double* __restrict__ kinv, int n,
                                                         const double* __restrict__ rhs, int64_t ncols,
                                                         double* __restrict__ out) {
    const int lane = threadIdx.x & 31;
    const int64_t gw = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const int64_t total = ncols * (int64_t)n;
    for (int64_t o = gw; o < total; o += ((int64_t)gridDim.x * blockDim.x) >> 5) {
        const int64_t c = o / n;
        const int r = (int)(o - c * n);
        const double* Kr = kinv + (int64_t)r * n;
        const double* x = rhs + c * n;
        double acc = 0.0;
        for (int q = lane; q < n; q += 32) acc += __ldg(Kr + q) * __ldg(x + q);
        acc = warp_sum(acc);
        if (lane == 0) out[o] = acc;
    }
}

}  // namespace tro

extern "C" int tro_kkt_apply_f64(const double* kinv, int32_t n, const double* rhs, int64_t ncols, double* out,
                                 void* stream) {
    if (!kinv || !rhs || !out || n <= 0 || ncols < 0) return TRO_EINVAL;
    if (ncols == 0) return 0;
    cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
    if (n <= tro::kSmemMaxN) {
        const size_t smem = ((size_t)n * n + (size_t)tro::kTileCols * (n + 1)) * sizeof(double);
        if (smem > 48 * 1024) {
            cudaFuncSetAttribute(tro::kkt_apply_small, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        }
        const int64_t blocks = (ncols + tro::kTileCols - 1) / tro::kTileCols;
        tro::kkt_apply_small<<<(unsigned)blocks, 256, smem, st>>>(kinv, n, rhs, ncols, out);
    } else {
        int64_t warps = ncols * (int64_t)n;
        int64_t blocks = (warps + 7) / 8;
        if (blocks > 148 * 64) blocks = 148 * 64;
        tro::kkt_apply_large<<<(unsigned)blocks, 256, 0, st>>>(kinv, n, rhs, ncols, out);
    }
    return (int)cudaGetLastError();
}
