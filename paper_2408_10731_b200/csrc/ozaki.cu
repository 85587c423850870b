// Multi-agent QP step (solver_multiagent.py:156-165, 266-269) on the 5th-generation tensor cores:
// fp64 D = K_L^-1[0:nv, 0:nk] x R[nk x 3P] as an Ozaki-sliced int8 GEMM (tcgen05.mma kind::i8, TMEM
// accumulators, operands brought in by tensor-map TMA).
//
// Why int8: tcgen05 has no fp64 kind (ptxas rejects .kind::f64 for sm_100a) and TF32 is far too coarse
// for saddle inverses with cond ~1e11.  Ozaki's splitting makes the products EXACT:
//   A[r][k] = 2^ea(r) sum_i a_i[r][k] 128^-(i+1),  R[k][c] = 2^eb(c) sum_j b_j[k][c] 128^-(j+1)
// with int8 slices |a_i|, |b_j| <= 127 (row / column scaled, truncated 7 bits at a time, exactly in fp64), so
//   D[r][c] = 2^(ea + eb) sum_d 128^-(d+2) P_d[r][c],   P_d = sum_{i+j=d} sum_k a_i b_j   (exact in int32:
// (d+1) nk 127^2 < 2^31).  Keeping the pairs with d < S drops terms below 128^-(S+1) relative to
// sum_k |A||R| (S = 7: ~1e-17), so the result is the exactly rounded-to-fp64 sum of the exact products up
// to that truncation: better than an fp64 FMA chain (DMMA), whose error grows with nk.
//
// The K dimension is two blocks with their own exponents: the primal columns [0, nv) (against rho B - C,
// large) and the boundary columns [nv, nk) (against b_eq, O(1)); one exponent over both would bound the error
// by max|A_r| max|R_c|, which the saddle inverse's structure makes ~1e4 x larger than the result.
//
// Kernel: persistent, one CTA per SM over (128-row m-tile, 32-column n-tile) tiles; warp 0 = TMA producer (2-D tensor maps over
// the pre-tiled int8 slices: every (slice, tile, k-step) operand is one 4 KB / 1 KB box already in the
// canonical no-swizzle K-major core-matrix layout), warp 1 = TMEM allocator + MMA issuer (one elected lane:
// S(S+1)/2 MMAs of 128x32x32 per k-step into 2 x S int32 accumulators of 32 TMEM columns each), warps 4-11 =
// epilogue (tcgen05.ld 32x32b, Horner in fp64, exact power-of-two scaling, coalesced xi stores).  Columns of
// problems at different rho levels: one pass per level present in the tile (A slices are per level; the
// B slices carry each column's own rho).
#include <cuda.h>
#include <cudaTypedefs.h>
#include <cuda_runtime.h>
#include <stdint.h>

#include "common.cuh"
#include "tma.cuh"
#include "../../include/trajopt_b200.h"

namespace tro {
namespace oz {

constexpr int BM = 128, BN = 32, BK = 32;  // one tcgen05.mma.kind::i8: M 128, N 32, K 32
constexpr int kABytes = BM * BK;           // 4096: one (slice, m-tile, k-step) A operand
constexpr int kBBytes = BN * BK;           // 1024: one (slice, n-tile, k-step) B operand
constexpr int kStages = 3;
constexpr int kMaxKs = 16;                 // nk <= 512
constexpr int kMaxMt = 2;                  // nv <= 256

// canonical no-swizzle K-major layout of an R x 32 int8 operand: [R / 8 row groups][2 k-cores][8 rows][16 B]
// (core matrix = 8 rows x 16 bytes; LBO = 128 B between k-cores, SBO = 256 B between row groups)
__host__ __device__ inline int canon_off(int r, int k) { return (r >> 3) * 256 + (k >> 4) * 128 + (r & 7) * 16 + (k & 15); }

__device__ __forceinline__ uint64_t sdesc(uint32_t saddr) {
    uint64_t d = 0;
    d |= (uint64_t)((saddr >> 4) & 0x3FFFu);
    d |= (uint64_t)((128u >> 4) & 0x3FFFu) << 16;  // leading byte offset: next core matrix along K
    d |= (uint64_t)((256u >> 4) & 0x3FFFu) << 32;  // stride byte offset: next 8-row group along M / N
    d |= (uint64_t)1 << 46;                         // descriptor version (sm_100)
    return d;                                       // base offset 0, layout type 0 (no swizzle)
}

// instruction descriptor: D s32, A / B signed int8, both K-major, N 32, M 128
constexpr uint32_t kIdesc = (2u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)(BN >> 3) << 17) | ((uint32_t)(BM >> 4) << 24);

__device__ __forceinline__ void umma_i8(uint32_t tmem_d, uint64_t da, uint64_t db, uint32_t acc) {
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "setp.ne.b32 p, %3, 0;\n\t"
        "tcgen05.mma.cta_group::1.kind::i8 [%0], %1, %2, %4, p;\n\t}\n" ::"r"(tmem_d),
        "l"(da), "l"(db), "r"(acc), "r"(kIdesc));
}
__device__ __forceinline__ void umma_commit(uint64_t* bar) {
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"l"(
                     (uint64_t)__cvta_generic_to_shared(bar))
                 : "memory");
}
__device__ __forceinline__ void tc_fence_after() { asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory"); }
__device__ __forceinline__ void tc_fence_before() { asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory"); }

__device__ __forceinline__ void tma_2d(void* dst, const CUtensorMap* map, int x, int y, uint64_t* bar) {
    asm volatile(
        "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];" ::"r"(
            smem_u32(dst)),
        "l"((uint64_t)map), "r"(x), "r"(y), "r"(smem_u32(bar))
        : "memory");
}

// 8 consecutive 32-bit TMEM columns of this thread's lane
__device__ __forceinline__ void tmem_ld8(uint32_t taddr, int32_t* v) {
    asm volatile("tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0, %1, %2, %3, %4, %5, %6, %7}, [%8];"
                 : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7])
                 : "r"(taddr));
}
__device__ __forceinline__ void tmem_wait_ld() { asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory"); }

struct OzArgs {
    int nv, nk, ks0, ks1, mt, nt;  // rows, K, k-steps of the primal / boundary K blocks, m-tiles, n-tiles
    int n_problems, n_agents, m, n_eq, n_levels;
    const int32_t* level;
    const int32_t* status;
    const int32_t* a_exp;  // n_levels x 2 x (mt * 128)
    const int32_t* b_exp;  // 2 x nt * 32
    double* xi;            // B x 3 x nv
};

// 2^e as a double, built from the exponent field (e within the normal range)
__device__ __forceinline__ double pow2(int e) {
    e = max(-1022, min(1023, e));
    return __longlong_as_double((long long)(e + 1023) << 52);
}

// ---------------------------------------------------------------- B slices: R columns -> int8 slices
// one warp per column c = 3 p + ax: R[k][c] = rho_L sums_B - sums_C (k < nv: the primal K block),
// b_eq (nv <= k < nk: the boundary K block); per block a column exponent (max |R| < 2^eb) and S truncated
// 7-bit slices written in the tiled canonical layout [slice][n-tile][k-step][1024 B block], four consecutive
// k per 32-bit store; the boundary block's k-steps follow the primal block's (ks0 .. ks0 + ks1)
template <int S>
__global__ void __launch_bounds__(256) ozaki_split_b_kernel(tro_ma_dims d, tro_ma_consts c, tro_ma_state s,
                                                            int8_t* __restrict__ bs, int32_t* __restrict__ bexp,
                                                            int nt, int ks0, int ks1) {
    const int lane = threadIdx.x & 31;
    const int col = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
    const int N = nt * BN;
    if (col >= N) return;
    const int n_a = d.n_agents, m = d.m, nv = n_a * m, neq = d.n_eq, ks = ks0 + ks1;
    const int p = col / 3, ax = col - 3 * p;
    bool act = p < d.n_problems;
    int lv = 0;
    if (act) {
        act = !(s.status[p] & TRO_CONVERGED);
        lv = s.level[p];
    }
    const double rho = act ? c.level_rho[lv] : 0.0;
    const double* sg = s.sums + (int64_t)p * 2 * n_a * 3 * m;
    const int ntile = col / BN, n = col - ntile * BN;
    constexpr int kMaxG = (kMaxKs * BK / 4 + 31) / 32;
#pragma unroll
    for (int blk = 0; blk < 2; ++blk) {
        const int kb = blk ? neq : nv, kpb = (blk ? ks1 : ks0) * BK, kst0 = blk ? ks0 : 0;
        // this lane's k-groups g = lane + 32 u of the block (k = 4 g .. 4 g + 3)
        double v[kMaxG][4];
        double mx = 0.0;
#pragma unroll
        for (int u = 0; u < kMaxG; ++u) {
#pragma unroll
            for (int q = 0; q < 4; ++q) {
                const int k = 4 * (lane + 32 * u) + q;
                double x = 0.0;
                if (act && k < kb) {
                    if (!blk) {
                        const int a = k / m, cc = k - a * m;
                        const int o = (a * 3 + ax) * m + cc;
                        x = rho * sg[o] - sg[n_a * 3 * m + o];
                    } else {
                        x = c.b_eq[(int64_t)p * 3 * neq + ax * neq + k];
                    }
                }
                v[u][q] = x;
                mx = fmax(mx, fabs(x));
            }
        }
        mx = warp_max(mx);
        int e = 0;
        if (mx > 0.0) frexp(mx, &e);  // mx < 2^e
        if (lane == 0) bexp[blk * N + col] = e;
        const double sc = pow2(-e);
#pragma unroll
        for (int u = 0; u < kMaxG; ++u) {
            const int g = lane + 32 * u;
            if (4 * g >= kpb) break;
            double x[4];
#pragma unroll
            for (int q = 0; q < 4; ++q) x[q] = v[u][q] * sc;  // |x| < 1, exact
            const int k0 = 4 * g, kst = k0 / BK;
            const int off = canon_off(n, k0 - kst * BK);
#pragma unroll
            for (int i = 0; i < S; ++i) {
                uint32_t w = 0;
#pragma unroll
                for (int q = 0; q < 4; ++q) {
                    const double y = x[q] * 128.0;
                    const double t = trunc(y);
                    x[q] = y - t;  // exact
                    w |= (uint32_t)(uint8_t)(int8_t)(int)t << (8 * q);
                }
                int8_t* dst = bs + (((int64_t)i * nt + ntile) * ks + kst0 + kst) * kBBytes + off;
                *reinterpret_cast<uint32_t*>(dst) = w;
            }
        }
    }
}

// ---------------------------------------------------------------- the int8 GEMM + fp64 epilogue
// rho levels present among the active problems of columns [c0, c0 + BN): one GEMM pass each
__device__ __forceinline__ uint32_t tile_levels(const OzArgs& a, int c0) {
    uint32_t mask = 0;
    const int p0 = c0 / 3, p1 = min((c0 + BN - 1) / 3, a.n_problems - 1);
    for (int p = p0; p <= p1; ++p)
        if (!(a.status[p] & TRO_CONVERGED)) mask |= 1u << a.level[p];
    return mask;
}

// Persistent: one CTA per SM walks the tiles t = blockIdx.x, += gridDim.x (m-tile fastest, so the CTAs in
// flight share the level's A slices in L2).  The producer runs ahead across tiles (the stage ring never
// drains), the MMA warp starts a tile's MMAs as soon as the epilogue has emptied TMEM, and the epilogue of
// one tile overlaps the TMA loads of the next.
template <int S>
__global__ void __launch_bounds__(384, 1) ozaki_gemm_kernel(const __grid_constant__ CUtensorMap tmA,
                                                            const __grid_constant__ CUtensorMap tmB, OzArgs a) {
    extern __shared__ __align__(1024) unsigned char smraw[];
    constexpr int kStageBytes = S * (kABytes + kBBytes);
    unsigned char* stages = smraw;
    uint64_t* full = reinterpret_cast<uint64_t*>(smraw + kStages * kStageBytes);
    uint64_t* empty = full + kStages;
    uint64_t* tfull = empty + kStages;
    uint64_t* tempty = tfull + 1;
    uint32_t* tbase = reinterpret_cast<uint32_t*>(tempty + 1);

    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int n_tiles = a.nt * a.mt;
    const int ks = a.ks0 + a.ks1;
    static_assert(BN == 32, "the epilogue maps one column per lane");

    if (threadIdx.x == 0) {
        for (int s = 0; s < kStages; ++s) {
            mbar_init(&full[s], 1);
            mbar_init(&empty[s], 1);
        }
        mbar_init(tfull, 1);
        mbar_init(tempty, 256);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    if (warp == 1) {  // TMEM: 2 K blocks x S accumulators x 32 columns (512 allocated)
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(smem_u32(tbase)));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem = *tbase;

    if (warp == 0) {
        // ======================= TMA producer
        if (lane == 0) {
            int s = 0;
            uint32_t ph = 0;
            for (int tile = blockIdx.x; tile < n_tiles; tile += gridDim.x) {
                const int mt = tile % a.mt, nt = tile / a.mt;
                for (uint32_t lm = tile_levels(a, nt * BN); lm; lm &= lm - 1) {
                    const int L = __ffs(lm) - 1;
                    for (int kst = 0; kst < ks; ++kst) {
                        mbar_wait(&empty[s], ph ^ 1u);
                        unsigned char* st = stages + s * kStageBytes;
                        mbar_expect_tx(&full[s], kStageBytes);
                        for (int i = 0; i < S; ++i)
                            tma_2d(st + i * kABytes, &tmA, 0, (((L * S + i) * a.mt + mt) * ks + kst) * (kABytes / 256),
                                   &full[s]);
                        for (int j = 0; j < S; ++j)
                            tma_2d(st + S * kABytes + j * kBBytes, &tmB, 0, ((j * a.nt + nt) * ks + kst) * (kBBytes / 256),
                                   &full[s]);
                        if (++s == kStages) {
                            s = 0;
                            ph ^= 1u;
                        }
                    }
                }
            }
        }
    } else if (warp == 1) {
        // ======================= MMA issuer (one elected lane)
        int s = 0;
        uint32_t ph = 0;
        int pass = 0;
        for (int tile = blockIdx.x; tile < n_tiles; tile += gridDim.x) {
            const int nt = tile / a.mt;
            for (uint32_t lm = tile_levels(a, nt * BN); lm; lm &= lm - 1, ++pass) {
                if (pass > 0) mbar_wait(tempty, (uint32_t)((pass - 1) & 1));  // the epilogue drained TMEM
                tc_fence_after();
                for (int kst = 0; kst < ks; ++kst) {
                    mbar_wait(&full[s], ph);
                    tc_fence_after();
                    if (lane == 0) {
                        const uint32_t sa = smem_u32(stages + s * kStageBytes);
                        const uint32_t sb = sa + S * kABytes;
                        const int blk = kst < a.ks0 ? 0 : 1;
                        const bool first = kst == 0 || kst == a.ks0;  // first k-step of this K block
                        const uint32_t tb = tmem + blk * S * BN;
#pragma unroll
                        for (int dd = 0; dd < S; ++dd)
#pragma unroll
                            for (int i = 0; i <= dd; ++i)
                                umma_i8(tb + dd * BN, sdesc(sa + i * kABytes), sdesc(sb + (dd - i) * kBBytes),
                                        (!first || i > 0) ? 1u : 0u);
                        umma_commit(&empty[s]);  // frees the stage when these MMAs have read it
                    }
                    __syncwarp();
                    if (++s == kStages) {
                        s = 0;
                        ph ^= 1u;
                    }
                }
                if (lane == 0) umma_commit(tfull);  // accumulators complete
                __syncwarp();
            }
        }
    } else if (warp >= 4) {
        // ======================= epilogue: TMEM -> fp64 -> xi (8 warps: two per TMEM lane quarter, each
        // draining half of the tile's columns, so the single TMEM buffer is back to the MMA warp sooner)
        const int q = warp & 3;            // TMEM lane quarter of this warp
        const int half = (warp - 4) >> 2;  // which 16 columns
        const uint32_t tq = tmem + ((uint32_t)(32 * q) << 16);
        int pass = 0;
        for (int tile = blockIdx.x; tile < n_tiles; tile += gridDim.x) {
            const int mt = tile % a.mt, nt = tile / a.mt, c0 = nt * BN;
            const int row = mt * BM + 32 * q + lane;  // output row of K^-1
            // lane l holds column c0 + l's level and power-of-two scales (read while the MMAs run)
            const int my_col = c0 + lane;
            const int my_p = my_col / 3;
            int my_lv = -1;
            if (my_p < a.n_problems && !(a.status[my_p] & TRO_CONVERGED)) my_lv = a.level[my_p];
            const double my_s0 = pow2(a.b_exp[my_col] - 14), my_s1 = pow2(a.b_exp[a.nt * BN + my_col] - 14);
            for (uint32_t lm = tile_levels(a, c0); lm; lm &= lm - 1, ++pass) {
                const int L = __ffs(lm) - 1;
                const double sa0 = row < a.nv ? pow2(a.a_exp[(L * 2 + 0) * a.mt * BM + row]) : 0.0;
                const double sa1 = row < a.nv ? pow2(a.a_exp[(L * 2 + 1) * a.mt * BM + row]) : 0.0;
                mbar_wait(tfull, (uint32_t)(pass & 1));
                tc_fence_after();
#pragma unroll 1
                for (int cc = half * (BN / 2); cc < (half + 1) * (BN / 2); cc += 8) {
                    int32_t P[2][S][8];
#pragma unroll
                    for (int bl = 0; bl < 2; ++bl)
#pragma unroll
                        for (int dd = 0; dd < S; ++dd) tmem_ld8(tq + (bl * S + dd) * BN + cc, P[bl][dd]);
                    tmem_wait_ld();
#pragma unroll
                    for (int jj = 0; jj < 8; ++jj) {
                        const int cl = cc + jj, col = c0 + cl;
                        const int lv = __shfl_sync(0xffffffffu, my_lv, cl);
                        const double s0 = __shfl_sync(0xffffffffu, my_s0, cl);
                        const double s1 = __shfl_sync(0xffffffffu, my_s1, cl);
                        if (row >= a.nv || lv != L) continue;
                        const int p = col / 3, ax = col - 3 * p;
                        double v0 = (double)P[0][S - 1][jj], v1 = (double)P[1][S - 1][jj];  // Horner over 128^-d
#pragma unroll
                        for (int dd = S - 2; dd >= 0; --dd) {
                            v0 = fma(v0, 0.0078125, (double)P[0][dd][jj]);
                            v1 = fma(v1, 0.0078125, (double)P[1][dd][jj]);
                        }
                        // exact power-of-two scalings (no under/overflow at these magnitudes), one rounding each
                        a.xi[(int64_t)p * 3 * a.nv + ax * a.nv + row] = (v0 * s0) * sa0 + (v1 * s1) * sa1;
                    }
                }
                tc_fence_before();
                mbar_arrive(tempty);
            }
        }
    }
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    if (warp == 1) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tmem));
}

// ---------------------------------------------------------------- host: tensor maps
static PFN_cuTensorMapEncodeTiled_v12000 encode_fn() {
    static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
    if (!fn) {
        void* p = nullptr;
        cudaDriverEntryPointQueryResult q;
        if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
            q == cudaDriverEntryPointSuccess)
            fn = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(p);
    }
    return fn;
}

// a 2-D uint8 view [rows][256 B] of a tiled slice array; boxes of box_rows x 256 B (one operand block)
static int make_map(CUtensorMap* map, const void* base, uint64_t bytes, uint32_t box_rows) {
    auto fn = encode_fn();
    if (!fn) return (int)cudaErrorNotSupported;
    const cuuint64_t dims[2] = {256, bytes / 256};
    const cuuint64_t strides[1] = {256};
    const cuuint32_t box[2] = {256, box_rows};
    const cuuint32_t estr[2] = {1, 1};
    const CUresult r = fn(map, CU_TENSOR_MAP_DATA_TYPE_UINT8, 2, const_cast<void*>(base), dims, strides, box, estr,
                          CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                          CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    return r == CUDA_SUCCESS ? 0 : (int)cudaErrorInvalidValue;
}

template <int S>
static int run(const tro_ma_dims* d, const tro_ma_consts* c, const tro_ma_state* s, const tro_ozaki_ws* w,
               cudaStream_t st) {
    const int nv = d->n_agents * d->m, nk = nv + d->n_eq;
    const int ks0 = (nv + BK - 1) / BK, ks1 = (d->n_eq + BK - 1) / BK, ks = ks0 + ks1, mt = (nv + BM - 1) / BM;
    const int N = 3 * d->n_problems, nt = (N + BN - 1) / BN;
    if (ks0 > kMaxKs || ks1 > kMaxKs || mt > kMaxMt || w->n_col_tiles < nt || 2 * S * BN > 512) return TRO_EINVAL;
    // 1. B slices of every column
    {
        const int cols_per_block = 8;
        ozaki_split_b_kernel<S><<<(nt * BN + cols_per_block - 1) / cols_per_block, 32 * cols_per_block, 0, st>>>(
            *d, *c, *s, w->b_slices, w->b_exp, nt, ks0, ks1);
        const int rc = (int)cudaGetLastError();
        if (rc) return rc;
    }
    // 2. the GEMM
    CUtensorMap mA, mB;
    int rc = make_map(&mA, w->a_slices, (uint64_t)d->n_levels * S * mt * ks * kABytes, kABytes / 256);
    if (rc) return rc;
    rc = make_map(&mB, w->b_slices, (uint64_t)S * nt * ks * kBBytes, kBBytes / 256);
    if (rc) return rc;
    OzArgs a;
    a.nv = nv;
    a.nk = nk;
    a.ks0 = ks0;
    a.ks1 = ks1;
    a.mt = mt;
    a.nt = nt;
    a.n_problems = d->n_problems;
    a.n_agents = d->n_agents;
    a.m = d->m;
    a.n_eq = d->n_eq;
    a.n_levels = d->n_levels;
    a.level = s->level;
    a.status = s->status;
    a.a_exp = w->a_exp;
    a.b_exp = w->b_exp;
    a.xi = s->xi;
    const size_t smem = (size_t)kStages * S * (kABytes + kBBytes) + 1024;
    static bool attr[64] = {false};
    int dev = 0;
    cudaGetDevice(&dev);
    if (dev >= 0 && dev < 64 && !attr[dev]) {
        cudaFuncSetAttribute(ozaki_gemm_kernel<S>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        attr[dev] = true;
    }
    static int n_sm = 0;
    if (!n_sm) cudaDeviceGetAttribute(&n_sm, cudaDevAttrMultiProcessorCount, dev);
    const int tiles = nt * mt;
    ozaki_gemm_kernel<S><<<tiles < n_sm ? tiles : n_sm, 384, smem, st>>>(mA, mB, a);
    return (int)cudaGetLastError();
}

}  // namespace oz
}  // namespace tro

extern "C" int tro_ma_qp_ozaki(const tro_ma_dims* d, const tro_ma_consts* c, const tro_ma_state* s,
                               const tro_ozaki_ws* w, void* stream) {
    if (!d || !c || !s || !w || !w->a_slices || !w->a_exp || !w->b_slices || !w->b_exp) return TRO_EINVAL;
    if (d->n_levels < 1 || d->n_levels > 32) return TRO_EINVAL;
    if (d->n_problems <= 0) return 0;
    cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
    switch (w->n_slices) {
        case 6: return tro::oz::run<6>(d, c, s, w, st);
        case 7: return tro::oz::run<7>(d, c, s, w, st);
        case 8: return tro::oz::run<8>(d, c, s, w, st);
        default: return TRO_EINVAL;
    }
}
