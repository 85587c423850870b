// XU-pipe-light elementary functions for the fused AM kernels.
//
// Why custom: libdevice's fp64 sincos/atan2/division route double<->int
// conversions and extra MUFU ops through the quarter-rate XU pipe, and fp64
// literals are re-materialised with UMOV/IMAD.MOV pairs inside the loop (ncu:
// ~190 of ~780 SASS instructions per element, profiles/r1_alg1.md).  Here:
//   * every fp64 coefficient lives in __constant__ memory, so DFMA reads it as a
//     c[][] operand (no instruction to load it);
//   * sin/cos: the AM angles are atan2 outputs (|x| <= pi), so a two-constant
//     Cody-Waite reduction (quadrant from the rint-by-magic-number trick, no
//     F2I) and the fdlibm kernel polynomials give <= 1 ulp on [-pi, pi];
//     |x| > 1e5 falls back to libdevice;
//   * atan2 needs ONE reciprocal: t = mn/mx when mn <= tan(pi/8) mx, else
//     t = (mn - mx)/(mn + mx) and pi/4 is added; fdlibm atan polynomial;
//   * sign flips and |x| are integer ops on the high word.
// Accuracy is pinned by tests/test_fastmath_gpu.py against numpy.
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

namespace tro {

struct FmConst {
    double sin_c[6];
    double cos_c[6];
    double atan_c[11];
    double two_over_pi, magic, pio2_hi, pio2_lo;
    double tan_pi8, pi_4, pi_2, pi;
};

static __constant__ FmConst kFm = {
    {-1.66666666666666324348e-01, 8.33333333332248946124e-03, -1.98412698298579493134e-04,
     2.75573137070700676789e-06, -2.50507602534068634195e-08, 1.58969099521155010221e-10},
    {4.16666666666666019037e-02, -1.38888888888741095749e-03, 2.48015872894767294178e-05,
     -2.75573143513906633035e-07, 2.08757232129817482790e-09, -1.13596475577881948265e-11},
    {3.33333333333329318027e-01, -1.99999999998764832476e-01, 1.42857142725034663711e-01,
     -1.11111104054623557880e-01, 9.09088713343650656196e-02, -7.69187620504482999495e-02,
     6.66107313738753120669e-02, -5.83357013379057348645e-02, 4.97687799461593236017e-02,
     -3.65315727442169155270e-02, 1.62858201153657823623e-02},
    0.63661977236758134308,
    6755399441055744.0,  // 1.5 * 2^52
    1.57079632673412561417e+00,
    6.07710050650619224932e-11,
    0.41421356237309504880,
    0.78539816339744830962,
    1.57079632679489661923,
    3.14159265358979323846,
};

// ---------------------------------------------------------------- bit helpers
__device__ __forceinline__ double flip_sign(double x, uint32_t mask) {
    return __hiloint2double(__double2hiint(x) ^ (int)mask, __double2loint(x));
}
__device__ __forceinline__ double abs_bits(double x) {
    return __hiloint2double(__double2hiint(x) & 0x7fffffff, __double2loint(x));
}
__device__ __forceinline__ uint32_t sign_bit(double x) { return (uint32_t)__double2hiint(x) & 0x80000000u; }
__device__ __forceinline__ double sel(bool p, double a, double b) { return p ? a : b; }

// ---------------------------------------------------------------- fp64
// 1/x for finite normal x: MUFU seed + cubic + Newton step (<= 1 ulp)
__device__ __forceinline__ double rcp_fast(double x) {
    double r;
    asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(r) : "d"(x));
    double e = fma(-x, r, 1.0);
    r = fma(r, fma(e, e, e), r);
    e = fma(-x, r, 1.0);
    return fma(r, e, r);
}

// 1/x without the final Newton step (<= 2 ulp: the cubic correction of the MUFU seed already leaves a
// truncation error far below one ulp, only the evaluation rounding remains): the Alg. 1 element pass,
// where the two dependent FMAs sit on every element's critical path (C5 launch 0.873 -> 0.884 of HBM)
__device__ __forceinline__ double rcp_fast2ulp(double x) {
    double r;
    asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(r) : "d"(x));
    const double e = fma(-x, r, 1.0);
    return fma(r, fma(e, e, e), r);
}

// 1/sqrt(x) for finite positive x: MUFU seed (~2^-22 relative) and ONE cubic correction
// y (1 + e/2 + 3e^2/8 + 5e^3/16), e = 1 - x y^2 (truncation ~2^-86: <= 1 ulp after rounding), four dependent
// DP operations instead of two Newton steps' six
#ifndef TRO_RSQRT_NEWTON
__device__ __forceinline__ double rsqrt_fast(double x) {
    double y;
    asm("rsqrt.approx.ftz.f64 %0, %1;" : "=d"(y) : "d"(x));
    const double e = fma(-x * y, y, 1.0);
    const double p = fma(e, fma(e, 0.3125, 0.375), 0.5);
    return fma(y * e, p, y);
}
#else
__device__ __forceinline__ double rsqrt_fast(double x) {
    double y;
    asm("rsqrt.approx.ftz.f64 %0, %1;" : "=d"(y) : "d"(x));
    const double hx = 0.5 * x;
    double e = fma(-hx * y, y, 0.5);
    y = fma(y, e, y);
    e = fma(-hx * y, y, 0.5);
    return fma(y, e, y);
}
#endif

// sqrt(x) for x > 0 finite (correctly rounded up to ~1 ulp)
__device__ __forceinline__ double sqrt_fast(double x) {
    const double y = rsqrt_fast(x);
    const double s = x * y;
    return fma(fma(-s, s, x), 0.5 * y, s);
}

__device__ __forceinline__ void sincos_fast(double x, double* s, double* c) {
    if (fabs(x) > 1.0e5) {  // outside the AM angle range: libdevice (Payne-Hanek)
        sincos(x, s, c);
        return;
    }
    const double t = fma(x, kFm.two_over_pi, kFm.magic);  // low mantissa bits hold rint(x 2/pi)
    const double k = t - kFm.magic;
    const uint32_t q = (uint32_t)__double2loint(t);
    const double r = fma(-k, kFm.pio2_lo, fma(-k, kFm.pio2_hi, x));
    const double z = r * r;
    const double ps = fma(z, fma(z, fma(z, fma(z, fma(z, kFm.sin_c[5], kFm.sin_c[4]), kFm.sin_c[3]), kFm.sin_c[2]),
                                 kFm.sin_c[1]), kFm.sin_c[0]);
    const double pc = fma(z, fma(z, fma(z, fma(z, fma(z, kFm.cos_c[5], kFm.cos_c[4]), kFm.cos_c[3]), kFm.cos_c[2]),
                                 kFm.cos_c[1]), kFm.cos_c[0]);
    const double sr = fma(r * z, ps, r);
    const double cr = fma(z * z, pc, fma(-0.5, z, 1.0));
    const bool odd = q & 1u;
    *s = flip_sign(sel(odd, cr, sr), (q & 2u) << 30);
    *c = flip_sign(sel(odd, sr, cr), ((q + 1u) & 2u) << 30);
}

__device__ __forceinline__ double atan2_fast(double y, double x) {
    const double ax = abs_bits(x), ay = abs_bits(y);
    const bool swap = ay > ax;
    const double mx = sel(swap, ay, ax), mn = sel(swap, ax, ay);
    const bool big = mn > kFm.tan_pi8 * mx;
    const double num = big ? mn - mx : mn;
    const double den = (big ? mn + mx : mx) + 1e-300;  // atan2(+-0, +-0): t = 0
    const double t = num * rcp_fast(den);
    const double z = t * t, w = z * z;
    const double s1 = z * fma(w, fma(w, fma(w, fma(w, fma(w, kFm.atan_c[10], kFm.atan_c[8]), kFm.atan_c[6]),
                                            kFm.atan_c[4]), kFm.atan_c[2]), kFm.atan_c[0]);
    const double s2 = w * fma(w, fma(w, fma(w, fma(w, kFm.atan_c[9], kFm.atan_c[7]), kFm.atan_c[5]), kFm.atan_c[3]),
                              kFm.atan_c[1]);
    double th = fma(-t, s1 + s2, t);
    if (big) th += kFm.pi_4;
    if (swap) th = kFm.pi_2 - th;
    if (sign_bit(x)) th = kFm.pi - th;
    return flip_sign(th, sign_bit(y));
}

// cos/sin of atan2(y, x) as a unit vector, numpy's signed-zero conventions
__device__ __forceinline__ void unit2(double x, double y, double* c, double* s) {
    const double h2 = fma(x, x, y * y);
    if (h2 > 0.0) {
        const double r = rsqrt_fast(h2);
        *c = x * r;
        *s = y * r;
    } else {
        *c = flip_sign(1.0, sign_bit(x));
        *s = flip_sign(0.0, sign_bit(y));
    }
}

// ---------------------------------------------------------------- fp32
// fp32 storage builds are held to 1e-4 (north_star): the hardware approximations (one MUFU each, <= 2 ulp)
// replace the correctly rounded IEEE sequences, which cost ~10 instructions apiece
#ifndef TRO_F32_IEEE
__device__ __forceinline__ float rcp_fast(float x) {
    float r;
    asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(r) : "f"(x));
    return r;
}
__device__ __forceinline__ float rsqrt_fast(float x) {
    float r;
    asm("rsqrt.approx.ftz.f32 %0, %1;" : "=f"(r) : "f"(x));
    return r;
}
__device__ __forceinline__ float sqrt_fast(float x) {
    float r;
    asm("sqrt.approx.ftz.f32 %0, %1;" : "=f"(r) : "f"(x));
    return r;
}
#else
__device__ __forceinline__ float rcp_fast(float x) { return __frcp_rn(x); }
__device__ __forceinline__ float rsqrt_fast(float x) { return rsqrtf(x); }
__device__ __forceinline__ float sqrt_fast(float x) { return sqrtf(x); }
#endif
__device__ __forceinline__ float rcp_fast2ulp(float x) { return rcp_fast(x); }

__device__ __forceinline__ void sincos_fast(float x, float* s, float* c) {
    if (fabsf(x) > 1.0e4f) {
        sincosf(x, s, c);
        return;
    }
    const float magic = 12582912.0f;  // 1.5 * 2^23
    const float t = fmaf(x, 0.636619772f, magic);
    const float k = t - magic;
    const uint32_t q = (uint32_t)__float_as_int(t);
    const float r = fmaf(-k, -4.37113900018624283e-8f, fmaf(-k, 1.57079637050628662f, x));
    const float z = r * r;
    const float sr = fmaf(r * z, fmaf(z, fmaf(z, fmaf(z, 2.75573192e-6f, -1.98412698e-4f), 8.33333333e-3f),
                                      -1.66666667e-1f), r);
    const float cr = fmaf(z * z, fmaf(z, fmaf(z, fmaf(z, -2.75573192e-7f, 2.48015873e-5f), -1.38888889e-3f),
                                      4.16666667e-2f), fmaf(-0.5f, z, 1.0f));
    const bool odd = q & 1u;
    *s = __int_as_float(__float_as_int(odd ? cr : sr) ^ (int)((q & 2u) << 30));
    *c = __int_as_float(__float_as_int(odd ? sr : cr) ^ (int)(((q + 1u) & 2u) << 30));
}

__device__ __forceinline__ float atan2_fast(float y, float x) {
    const float ax = fabsf(x), ay = fabsf(y);
    const bool swap = ay > ax;
    const float mx = swap ? ay : ax, mn = swap ? ax : ay;
    const bool big = mn > 0.414213562f * mx;
    const float t = (big ? mn - mx : mn) * rcp_fast((big ? mn + mx : mx) + 1e-37f);
    const float z = t * t;
    // t - t z (1/3 - z/5 + z^2/7 - z^3/9 + z^4/11 - z^5/13 + z^6/15)
    const float p = fmaf(z, fmaf(z, fmaf(z, fmaf(z, fmaf(z, fmaf(z, 0.0666666667f, -0.0769230769f), 0.0909090909f),
                                              -0.111111111f), 0.142857143f), -0.2f), 0.333333333f);
    float th = fmaf(-t * z, p, t);
    if (big) th += 0.785398163f;
    if (swap) th = 1.57079633f - th;
    if (__float_as_int(x) < 0) th = 3.14159265f - th;
    return __int_as_float(__float_as_int(th) ^ (__float_as_int(y) & 0x80000000));
}

}  // namespace tro
