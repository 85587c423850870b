// Stable ascending top-k selection for CEM / PRIEST elites.
//
// Reference semantics: np.argsort(keys, kind="stable")[:k]
// (solver_priest.py:358, :440) — ascending, ties broken by index, NaN last,
// -0.0 == +0.0.  Bit-exact by construction: each key is mapped to an
// order-preserving uint64 and every comparison is on (u64 key, index) pairs;
// no floating-point arithmetic touches the keys, so the result is identical
// for any launch geometry or GPU count.
//
// Two paths:
//  * small n (<= kRankMaxN): exact-rank scatter, rank_i = #{ j : (u_j, j) < (u_i, i) }, one CTA per 256
//    candidates streaming the keys through shared memory (O(n^2) work, two launches: latency-optimal);
//  * large n: radix SELECT in O(n): eight MSD passes of 8-bit digits find the k-th smallest key T and how many
//    of its ties are taken (each pass: per-block shared-memory histograms, one global histogram, the last
//    block to finish picks the digit: no host round trip), a compaction pass writes the keys < T and the
//    first ties of T in index order (block prefix sums), and a bitonic sort of the k (key, index) pairs
//    (shared-memory stages for strides < 2048, global stages above) writes the indices in rank order:
//    O(n + k log^2 k).
#include "common.cuh"
#include "../../include/trajopt_b200.h"

namespace tro {

constexpr int kRankThreads = 256;
constexpr int kKeyTile = 2048;
constexpr int64_t kRankMaxN = 4096;

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

// ---------------------------------------------------------------- radix select
struct SelState {
    uint64_t prefix, mask;  // digits of T found so far
    int64_t kk;             // rank still to find inside the current prefix (1-based)
    uint32_t ticket;
    uint32_t hist[256];
};

constexpr int kSelThreads = 512;

__global__ void __launch_bounds__(kSelThreads) radix_pass(const uint64_t* __restrict__ u, int64_t n, int shift,
                                                          SelState* st) {
    __shared__ uint32_t h[256];
    __shared__ bool last;
    for (int b = threadIdx.x; b < 256; b += blockDim.x) h[b] = 0;
    __syncthreads();
    const uint64_t prefix = st->prefix, mask = st->mask;
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
        const uint64_t v = u[i];
        if ((v & mask) == prefix) atomicAdd(&h[(v >> shift) & 255u], 1u);
    }
    __syncthreads();
    for (int b = threadIdx.x; b < 256; b += blockDim.x)
        if (h[b]) atomicAdd(&st->hist[b], h[b]);
    __threadfence();
    __syncthreads();
    if (threadIdx.x == 0) last = atomicAdd(&st->ticket, 1u) == gridDim.x - 1;
    __syncthreads();
    if (!last) return;
    __threadfence();
    // the last block picks the digit: the global histogram into shared memory (parallel loads), then one
    // warp-wide inclusive scan of the 256 bins (8 per lane)
    for (int b = threadIdx.x; b < 256; b += blockDim.x) h[b] = ((volatile uint32_t*)st->hist)[b];
    __syncthreads();
    if (threadIdx.x < 32) {
        const int lane = threadIdx.x;
        const int64_t kk = st->kk;
        int64_t loc[8], run = 0;
#pragma unroll
        for (int q = 0; q < 8; ++q) {
            run += h[lane * 8 + q];
            loc[q] = run;
        }
        int64_t excl = run;  // inclusive scan of the lane totals
        for (int o = 1; o < 32; o <<= 1) {
            const int64_t x = __shfl_up_sync(0xffffffffu, excl, o);
            if (lane >= o) excl += x;
        }
        excl -= run;  // exclusive prefix of this lane's first bin
        // first bin whose inclusive cumulative count reaches kk
        int digit = 256;
#pragma unroll
        for (int q = 7; q >= 0; --q)
            if (excl + loc[q] >= kk) digit = lane * 8 + q;
        for (int o = 16; o > 0; o >>= 1) digit = min(digit, __shfl_xor_sync(0xffffffffu, digit, o));
        if (lane == digit / 8) {
            const int q = digit % 8;
            const int64_t before = excl + (q ? loc[q - 1] : 0);
            st->kk = kk - before;
            st->prefix = prefix | ((uint64_t)digit << shift);
            st->mask = mask | (0xFFull << shift);
            st->ticket = 0;
        }
    }
    __syncthreads();
    for (int b = threadIdx.x; b < 256; b += blockDim.x) st->hist[b] = 0;
}

__global__ void sel_init(SelState* st, int64_t k) {
    if (threadIdx.x == 0) {
        st->prefix = 0;
        st->mask = 0;
        st->kk = k;
        st->ticket = 0;
    }
    for (int b = threadIdx.x; b < 256; b += blockDim.x) st->hist[b] = 0;
}

constexpr int kCompBlock = 1024;  // elements per compaction block

// per block: (#keys < T, #keys == T)
__global__ void __launch_bounds__(kCompBlock) sel_count(const uint64_t* __restrict__ u, int64_t n,
                                                        const SelState* st, uint32_t* __restrict__ cnt) {
    const uint64_t T = st->prefix;
    const int64_t i = (int64_t)blockIdx.x * kCompBlock + threadIdx.x;
    const uint64_t v = i < n ? u[i] : ~0ull;
    const bool lt = i < n && v < T, eq = i < n && v == T;
    const uint32_t blt = __syncthreads_count(lt), beq = __syncthreads_count(eq);
    if (threadIdx.x == 0) {
        cnt[2 * blockIdx.x] = blt;
        cnt[2 * blockIdx.x + 1] = beq;
    }
}

// exclusive prefix over blocks (one CTA, sequential chunks)
__global__ void __launch_bounds__(1024) sel_scan(uint32_t* __restrict__ cnt, int nb) {
    __shared__ uint32_t carry[2];
    if (threadIdx.x == 0) carry[0] = carry[1] = 0;
    __syncthreads();
    for (int c0 = 0; c0 < nb; c0 += 1024) {
        const int b = c0 + threadIdx.x;
        uint32_t lt = b < nb ? cnt[2 * b] : 0, eq = b < nb ? cnt[2 * b + 1] : 0;
        // inclusive block scans of both counters
        __shared__ uint32_t s0[1024], s1[1024];
        s0[threadIdx.x] = lt;
        s1[threadIdx.x] = eq;
        __syncthreads();
        for (int o = 1; o < 1024; o <<= 1) {
            const uint32_t a0 = threadIdx.x >= o ? s0[threadIdx.x - o] : 0, a1 = threadIdx.x >= o ? s1[threadIdx.x - o] : 0;
            __syncthreads();
            s0[threadIdx.x] += a0;
            s1[threadIdx.x] += a1;
            __syncthreads();
        }
        if (b < nb) {
            cnt[2 * b] = carry[0] + s0[threadIdx.x] - lt;
            cnt[2 * b + 1] = carry[1] + s1[threadIdx.x] - eq;
        }
        __syncthreads();
        if (threadIdx.x == 1023) {
            carry[0] += s0[1023];
            carry[1] += s1[1023];
        }
        __syncthreads();
    }
}

// keys < T go to slots [0, k - kk) in index order, the first kk ties of T to [k - kk, k)
__global__ void __launch_bounds__(kCompBlock) sel_write(const uint64_t* __restrict__ u, int64_t n, int64_t k,
                                                        const SelState* st, const uint32_t* __restrict__ off,
                                                        uint64_t* __restrict__ ck, uint64_t* __restrict__ ci) {
    __shared__ uint32_t w0[kCompBlock / 32], w1[kCompBlock / 32];
    const uint64_t T = st->prefix;
    const int64_t n_lt = k - st->kk;
    const int64_t i = (int64_t)blockIdx.x * kCompBlock + threadIdx.x;
    const uint64_t v = i < n ? u[i] : ~0ull;
    const bool lt = i < n && v < T, eq = i < n && v == T;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const uint32_t b0 = __ballot_sync(0xffffffffu, lt), b1 = __ballot_sync(0xffffffffu, eq);
    if (lane == 0) {
        w0[warp] = __popc(b0);
        w1[warp] = __popc(b1);
    }
    __syncthreads();
    if (threadIdx.x < 32) {  // exclusive scan of the warp counts
        uint32_t a = w0[lane], c = w1[lane];
        for (int o = 1; o < 32; o <<= 1) {
            const uint32_t x = __shfl_up_sync(0xffffffffu, a, o), y = __shfl_up_sync(0xffffffffu, c, o);
            if (lane >= o) {
                a += x;
                c += y;
            }
        }
        w0[lane] = a - w0[lane];
        w1[lane] = c - w1[lane];
    }
    __syncthreads();
    const uint32_t below = (1u << lane) - 1u;
    if (lt) {
        const int64_t r = off[2 * blockIdx.x] + w0[warp] + __popc(b0 & below);
        ck[r] = v;
        ci[r] = (uint64_t)i;
    } else if (eq) {
        const int64_t r = off[2 * blockIdx.x + 1] + w1[warp] + __popc(b1 & below);
        if (r < st->kk) {
            ck[n_lt + r] = v;
            ci[n_lt + r] = (uint64_t)i;
        }
    }
}

// ---------------------------------------------------------------- bitonic sort of (key, index) pairs
constexpr int kBitLocal = 2048;  // pairs per shared-memory chunk

__device__ __forceinline__ bool pair_less(uint64_t ka, uint64_t ia, uint64_t kb, uint64_t ib) {
    return ka < kb || (ka == kb && ia < ib);
}

// pads [k, p2) with (max, max), then sorts every 2048-chunk (size < = 2048 stages)  when full = true, or only
// the merge stages of the given size for strides < 2048 (full = false)
__global__ void __launch_bounds__(1024) bitonic_local(uint64_t* __restrict__ ck, uint64_t* __restrict__ ci,
                                                      int64_t k, int64_t p2, int64_t size, bool full) {
    __shared__ uint64_t sk[kBitLocal], si[kBitLocal];
    const int64_t base = (int64_t)blockIdx.x * kBitLocal;
    for (int q = threadIdx.x; q < kBitLocal; q += blockDim.x) {
        const int64_t g = base + q;
        const bool pad = g >= k;
        sk[q] = pad ? ~0ull : ck[g];
        si[q] = pad ? ~0ull : ci[g];
    }
    __syncthreads();
    const int64_t s0 = full ? 2 : size, s1 = full ? (p2 < kBitLocal ? p2 : kBitLocal) : size;
    for (int64_t sz = s0; sz <= s1; sz <<= 1) {
        for (int64_t j = (sz >> 1) < (kBitLocal >> 1) ? (sz >> 1) : (kBitLocal >> 1); j > 0; j >>= 1) {
            for (int q = threadIdx.x; q < kBitLocal; q += blockDim.x) {
                const int r = q ^ (int)j;
                if (r > q) {
                    const bool up = ((base + q) & sz) == 0;
                    const bool sw = pair_less(sk[r], si[r], sk[q], si[q]) == up;
                    if (sw) {
                        const uint64_t tk = sk[q], ti = si[q];
                        sk[q] = sk[r];
                        si[q] = si[r];
                        sk[r] = tk;
                        si[r] = ti;
                    }
                }
            }
            __syncthreads();
        }
    }
    for (int q = threadIdx.x; q < kBitLocal; q += blockDim.x) {
        ck[base + q] = sk[q];
        ci[base + q] = si[q];
    }
}

__global__ void bitonic_global(uint64_t* __restrict__ ck, uint64_t* __restrict__ ci, int64_t p2, int64_t size,
                               int64_t j) {
    for (int64_t q = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; q < p2; q += (int64_t)gridDim.x * blockDim.x) {
        const int64_t r = q ^ j;
        if (r > q) {
            const bool up = (q & size) == 0;
            if (pair_less(ck[r], ci[r], ck[q], ci[q]) == up) {
                const uint64_t tk = ck[q], ti = ci[q];
                ck[q] = ck[r];
                ci[q] = ci[r];
                ck[r] = tk;
                ci[r] = ti;
            }
        }
    }
}

__global__ void write_out(const uint64_t* __restrict__ ci, int64_t k, int64_t* __restrict__ out) {
    for (int64_t q = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; q < k; q += (int64_t)gridDim.x * blockDim.x)
        out[q] = (int64_t)ci[q];
}

__host__ __device__ inline int64_t pow2_at_least(int64_t x, int64_t lo) {
    int64_t p = lo;
    while (p < x) p <<= 1;
    return p;
}

// workspace: u (n) | state | block counts (2 nb) | candidate keys (p2) | candidate indices (p2)
struct TopkWs {
    uint64_t* u;
    SelState* st;
    uint32_t* cnt;
    uint64_t* ck;
    uint64_t* ci;
    int64_t bytes;
};
__host__ __device__ inline TopkWs topk_ws(void* base, int64_t n, int64_t k) {
    TopkWs w;
    unsigned char* p = reinterpret_cast<unsigned char*>(base);
    int64_t off = 0;
    w.u = reinterpret_cast<uint64_t*>(p + off);
    off += n * 8;
    if (n <= kRankMaxN) {
        w.st = nullptr;
        w.cnt = nullptr;
        w.ck = w.ci = nullptr;
        w.bytes = off;
        return w;
    }
    off = (off + 255) & ~(int64_t)255;
    w.st = reinterpret_cast<SelState*>(p + off);
    off += (int64_t)sizeof(SelState);
    off = (off + 255) & ~(int64_t)255;
    const int64_t nb = (n + kCompBlock - 1) / kCompBlock;
    w.cnt = reinterpret_cast<uint32_t*>(p + off);
    off += 2 * nb * 4;
    off = (off + 255) & ~(int64_t)255;
    const int64_t p2 = pow2_at_least(k, kBitLocal);
    w.ck = reinterpret_cast<uint64_t*>(p + off);
    off += p2 * 8;
    w.ci = reinterpret_cast<uint64_t*>(p + off);
    off += p2 * 8;
    w.bytes = off;
    return w;
}

}  // namespace tro

extern "C" int64_t tro_topk_workspace_bytes(int64_t n, int32_t k) {
    if (n <= 0) return 0;
    return tro::topk_ws(nullptr, n, k > 0 ? k : 1).bytes;
}

extern "C" int tro_topk_stable_f64(const double* keys, int64_t n, int32_t k, int64_t* out_idx, void* workspace,
                                   int64_t workspace_bytes, void* stream) {
    if (n < 0 || k < 0 || k > n) return TRO_EINVAL;
    if (n == 0 || k == 0) return 0;
    if (!keys || !out_idx || !workspace || workspace_bytes < tro_topk_workspace_bytes(n, k)) return TRO_EINVAL;
    cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
    const tro::TopkWs w = tro::topk_ws(workspace, n, k);
    int64_t blocks = (n + 255) / 256;
    if (blocks > 148 * 16) blocks = 148 * 16;
    tro::to_order_keys<<<(unsigned)blocks, 256, 0, st>>>(keys, n, w.u);
    if (n <= tro::kRankMaxN) {
        const int64_t rb = (n + tro::kRankThreads - 1) / tro::kRankThreads;
        tro::rank_scatter<<<(unsigned)rb, tro::kRankThreads, 0, st>>>(w.u, n, k, out_idx);
        return (int)cudaGetLastError();
    }
    // radix select of the k-th smallest key
    tro::sel_init<<<1, 256, 0, st>>>(w.st, k);
    int64_t hb = (n + tro::kSelThreads * 8 - 1) / (tro::kSelThreads * 8);
    if (hb > 148 * 4) hb = 148 * 4;
    for (int pass = 0; pass < 8; ++pass)
        tro::radix_pass<<<(unsigned)hb, tro::kSelThreads, 0, st>>>(w.u, n, 56 - 8 * pass, w.st);
    // compaction in index order
    const int64_t nb = (n + tro::kCompBlock - 1) / tro::kCompBlock;
    tro::sel_count<<<(unsigned)nb, tro::kCompBlock, 0, st>>>(w.u, n, w.st, w.cnt);
    tro::sel_scan<<<1, 1024, 0, st>>>(w.cnt, (int)nb);
    tro::sel_write<<<(unsigned)nb, tro::kCompBlock, 0, st>>>(w.u, n, k, w.st, w.cnt, w.ck, w.ci);
    // bitonic sort of the k pairs (padded to a power of two >= 2048)
    const int64_t p2 = tro::pow2_at_least(k, tro::kBitLocal);
    const unsigned chunks = (unsigned)(p2 / tro::kBitLocal);
    tro::bitonic_local<<<chunks, 1024, 0, st>>>(w.ck, w.ci, k, p2, 0, true);
    for (int64_t size = 2 * tro::kBitLocal; size <= p2; size <<= 1) {
        for (int64_t j = size >> 1; j >= tro::kBitLocal; j >>= 1) {
            int64_t gb = (p2 + 255) / 256;
            if (gb > 148 * 16) gb = 148 * 16;
            tro::bitonic_global<<<(unsigned)gb, 256, 0, st>>>(w.ck, w.ci, p2, size, j);
        }
        tro::bitonic_local<<<chunks, 1024, 0, st>>>(w.ck, w.ci, p2, p2, size, false);
    }
    tro::write_out<<<(unsigned)((k + 255) / 256), 256, 0, st>>>(w.ci, k, out_idx);
    return (int)cudaGetLastError();
}
