// Library-level C entry points (version / error strings).
#include <cuda_runtime.h>
#include "../../include/trajopt_b200.h"

extern "C" int32_t tro_version(void) { return 1; }

extern "C" const char* tro_error_string(int32_t code) {
    if (code == 0) return "success";
    if (code == TRO_EINVAL) return "invalid argument (host-side check)";
    return cudaGetErrorString((cudaError_t)code);
}
