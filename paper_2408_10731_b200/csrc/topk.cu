// Stable ascending top-k selection for CEM / PRIEST elites.
//
// Reference semantics: np.argsort(keys, kind="stable")[:k]
// (solver_priest.py:358, :440) — ascending, ties broken by index, NaN last,
// -0.0 == +0.0.  Bit-exact by construction: each key is mapped to an
// order-preserving uint64, and element i's output slot is its exact rank
// rank_i = #{ j : (u_j, j) < (u_i, i) }; element i is an elite iff rank_i < k
// and is written to out[rank_i].  No floating-point arithmetic touches the
// keys, so the result is identical for any launch geometry or GPU count.
//
// Each CTA ranks 256 candidates against all keys streamed through shared
// memory in tiles (broadcast reads, no bank conflicts); a warp-level ballot
// skips tiles that cannot change any candidate's rank.
#include "common.cuh"
#include "../../include/trajopt_b200.h"

namespace tro {

constexpr int kRankThreads = 256;
constexpr int kKeyTile = 2048;

__device__ __forceinline__ uint64_t order_key(double x) {
    if (x != x) return 0xFFFFFFFFFFFFFFFFull;  // NaN sorts last
    if (x == 0.0) x = 0.0;                     // -0.0 ties with +0.0
    uint64_t u = (uint64_t)__double_as_longlong(x);
    return (u & 0x8000000000000000ull) ? ~u : (u | 0x8000000000000000ull);
}

__global__ void to_order_keys(const double* __restrict__ keys, int64_t n, uint64_t* __restrict__ u) {
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
        u[i] = order_key(keys[i]);
}

__global__ void __launch_bounds__(kRankThreads) rank_scatter(const uint64_t* __restrict__ u, int64_t n, int k,
                                                             int64_t* __restrict__ out) {
    __shared__ uint64_t tile[kKeyTile];
    const int64_t i = (int64_t)blockIdx.x * kRankThreads + threadIdx.x;
    const bool valid = i < n;
    const uint64_t ui = valid ? u[i] : 0xFFFFFFFFFFFFFFFFull;
    int64_t rank = 0;
    for (int64_t j0 = 0; j0 < n; j0 += kKeyTile) {
        const int cnt = (n - j0) < kKeyTile ? (int)(n - j0) : kKeyTile;
        __syncthreads();
        for (int q = threadIdx.x; q < cnt; q += kRankThreads) tile[q] = u[j0 + q];
        __syncthreads();
        if (valid) {
            int r = 0;
            if (j0 + cnt <= i) {
                // whole tile precedes i: ties count
#pragma unroll 8
                for (int q = 0; q < cnt; ++q) r += (tile[q] <= ui);
            } else if (j0 > i) {
                // whole tile follows i: only strictly smaller keys count
#pragma unroll 8
                for (int q = 0; q < cnt; ++q) r += (tile[q] < ui);
            } else {
                for (int q = 0; q < cnt; ++q) {
                    const int64_t j = j0 + q;
                    r += (tile[q] < ui) || (tile[q] == ui && j < i);
                }
            }
            rank += r;
        }
    }
    if (valid && rank < k) out[rank] = i;
}

}  // namespace tro

extern "C" int64_t tro_topk_workspace_bytes(int64_t n, int32_t k) {
    (void)k;
    return n > 0 ? n * (int64_t)sizeof(uint64_t) : 0;
}

extern "C" int tro_topk_stable_f64(const double* keys, int64_t n, int32_t k, int64_t* out_idx, void* workspace,
                                   int64_t workspace_bytes, void* stream) {
    if (n < 0 || k < 0 || k > n) return TRO_EINVAL;
    if (n == 0 || k == 0) return 0;
    if (!keys || !out_idx || !workspace || workspace_bytes < tro_topk_workspace_bytes(n, k)) return TRO_EINVAL;
    cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
    uint64_t* u = reinterpret_cast<uint64_t*>(workspace);
    int64_t blocks = (n + 255) / 256;
    if (blocks > 148 * 16) blocks = 148 * 16;
    tro::to_order_keys<<<(unsigned)blocks, 256, 0, st>>>(keys, n, u);
    const int64_t rb = (n + tro::kRankThreads - 1) / tro::kRankThreads;
    tro::rank_scatter<<<(unsigned)rb, tro::kRankThreads, 0, st>>>(u, n, k, out_idx);
    return (int)cudaGetLastError();
}
