// Library-level C entry points (version / error strings).
#include <cuda_runtime.h>
#include "../../include/trajopt_b200.h"

extern "C" int32_t tro_version(void) { return 1; }

extern "C" const char* tro_error_string(int32_t code) {
    if (code == 0) return "success";
    if (code == TRO_EINVAL) return "invalid argument (host-side check)";
    return cudaGetErrorString((cudaError_t)code);
}

// FP64 FMA throughput probe (diagnostics): 8 independent DFMA chains per thread.
__global__ void fp64_peak_kernel(int64_t iters, double* out) {
    double a[8];
#pragma unroll
    for (int k = 0; k < 8; ++k) a[k] = 1.0 + 1e-9 * (threadIdx.x + k);
    const double b = 0.999999999, c = 1e-9;
    for (int64_t i = 0; i < iters; ++i) {
#pragma unroll
        for (int k = 0; k < 8; ++k) a[k] = fma(a[k], b, c);
    }
    double s = 0.0;
#pragma unroll
    for (int k = 0; k < 8; ++k) s += a[k];
    if (s == 12345.0) out[threadIdx.x] = s;  // keeps the chains alive
}

extern "C" int tro_fp64_fma_probe(int64_t iters, int32_t blocks, double* scratch, void* stream) {
    if (iters < 1 || blocks < 1 || !scratch) return TRO_EINVAL;
    fp64_peak_kernel<<<blocks, 256, 0, reinterpret_cast<cudaStream_t>(stream)>>>(iters, scratch);
    return (int)cudaGetLastError();
}
