// XU-pipe-free elementary functions for the fused AM kernels.
//
// libdevice's fp64 sincos/atan2/division spend double->int conversions and
// MUFU ops on the quarter-rate XU pipe; ncu showed that pipe as the limiter of
// the first fused kernel (profiles/r1_alg1_c2_baseline.md).  The angles of the
// AM iteration are atan2 outputs (|x| <= pi), so a two-constant Cody-Waite
// reduction plus the fdlibm kernel polynomials is exact enough (<= 1 ulp on
// [-pi, pi], checked against numpy in tests/test_fastmath.py), with a libdevice
// fallback for |x| > 1e5.  atan2 uses ONE reciprocal: t = mn/mx when
// mn <= tan(pi/8) mx, else t = (mn - mx)/(mn + mx) and pi/4 is added.
#pragma once
#include <cuda_runtime.h>

namespace tro {

// ---------------------------------------------------------------- fp64
__device__ __forceinline__ double rcp_fast(double x) {
    double r;
    asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(r) : "d"(x));
    double e = fma(-x, r, 1.0);
    r = fma(r, e, r);
    e = fma(-x, r, 1.0);
    r = fma(r, e, r);
    e = fma(-x, r, 1.0);
    return fma(r, e, r);
}

__device__ __forceinline__ double rsqrt_fast(double x) { return rsqrt(x); }

// fdlibm __kernel_sin / __kernel_cos on |r| <= pi/4
__device__ __forceinline__ void sincos_kernel(double r, double* s, double* c) {
    const double z = r * r;
    const double ps = fma(z, fma(z, fma(z, fma(z, fma(z, 1.58969099521155010221e-10, -2.50507602534068634195e-08),
                                                2.75573137070700676789e-06), -1.98412698298579493134e-04),
                                  8.33333333332248946124e-03), -1.66666666666666324348e-01);
    const double pc = fma(z, fma(z, fma(z, fma(z, fma(z, -1.13596475577881948265e-11, 2.08757232129817482790e-09),
                                                -2.75573143513906633035e-07), 2.48015872894767294178e-05),
                                  -1.38888888888741095749e-03), 4.16666666666666019037e-02);
    *s = fma(r * z, ps, r);
    *c = fma(z * z, pc, fma(-0.5, z, 1.0));
}

__device__ __forceinline__ void sincos_fast(double x, double* s, double* c) {
    if (fabs(x) > 1.0e5) {  // outside the AM angle range: libdevice (Payne-Hanek)
        sincos(x, s, c);
        return;
    }
    const double magic = 6755399441055744.0;  // 1.5 * 2^52: fma result's low mantissa bits hold rint()
    const double t = fma(x, 0.63661977236758134308, magic);
    const double k = t - magic;
    const int q = __double2loint(t) & 3;
    const double r = fma(-k, 6.07710050650619224932e-11, fma(-k, 1.57079632673412561417e+00, x));
    double sr, cr;
    sincos_kernel(r, &sr, &cr);
    const double ss = (q & 1) ? cr : sr;
    const double cc = (q & 1) ? sr : cr;
    *s = (q & 2) ? -ss : ss;
    *c = ((q + 1) & 2) ? -cc : cc;
}

// fdlibm atan polynomial on |t| <= tan(pi/8)
__device__ __forceinline__ double atan_kernel(double t) {
    const double z = t * t, w = z * z;
    const double s1 = z * fma(w, fma(w, fma(w, fma(w, fma(w, 1.62858201153657823623e-02, 4.97687799461593236017e-02),
                                                  6.66107313738753120669e-02), 9.09088713343650656196e-02),
                                      1.42857142725034663711e-01), 3.33333333333329318027e-01);
    const double s2 = w * fma(w, fma(w, fma(w, fma(w, -3.65315727442169155270e-02, -5.83357013379057348645e-02),
                                          -7.69187620504482999495e-02), -1.11111104054623557880e-01),
                              -1.99999999998764832476e-01);
    return fma(-t, s1 + s2, t);
}

__device__ __forceinline__ double atan2_fast(double y, double x) {
    const double ax = fabs(x), ay = fabs(y);
    const double mx = fmax(ax, ay), mn = fmin(ax, ay);
    if (!(mx > 0.0) || mx > 1.0e300 || mx != mx) return atan2(y, x);  // zeros / inf / nan: libdevice
    const bool big = mn > 0.41421356237309504880 * mx;
    const double num = big ? mn - mx : mn;
    const double den = big ? mn + mx : mx;
    const double t = num * rcp_fast(den);
    double th = atan_kernel(t);
    if (big) th += 0.78539816339744830962;
    if (ay > ax) th = 1.57079632679489661923 - th;
    if (x < 0.0) th = 3.14159265358979323846 - th;
    return copysign(th, y);
}

// ---------------------------------------------------------------- fp32
__device__ __forceinline__ float rcp_fast(float x) { return __frcp_rn(x); }
__device__ __forceinline__ float rsqrt_fast(float x) { return rsqrtf(x); }

__device__ __forceinline__ void sincos_fast(float x, float* s, float* c) {
    if (fabsf(x) > 1.0e4f) {
        sincosf(x, s, c);
        return;
    }
    const float magic = 12582912.0f;  // 1.5 * 2^23
    const float t = fmaf(x, 0.636619772f, magic);
    const float k = t - magic;
    const int q = __float_as_int(t) & 3;
    const float r = fmaf(-k, -4.37113900018624283e-8f, fmaf(-k, 1.57079637050628662f, x));
    const float z = r * r;
    const float sr = fmaf(r * z, fmaf(z, fmaf(z, fmaf(z, 2.75573137e-6f, -1.98412698e-4f), 8.33333333e-3f),
                                      -1.66666667e-1f), r);
    const float cr = fmaf(z * z, fmaf(z, fmaf(z, fmaf(z, 2.48015873e-5f * -0.0111111111f, 2.48015873e-5f),
                                               -1.38888889e-3f), 4.16666667e-2f), fmaf(-0.5f, z, 1.0f));
    const float ss = (q & 1) ? cr : sr;
    const float cc = (q & 1) ? sr : cr;
    *s = (q & 2) ? -ss : ss;
    *c = ((q + 1) & 2) ? -cc : cc;
}

__device__ __forceinline__ float atan2_fast(float y, float x) {
    const float ax = fabsf(x), ay = fabsf(y);
    const float mx = fmaxf(ax, ay), mn = fminf(ax, ay);
    if (!(mx > 0.0f) || mx > 1.0e30f || mx != mx) return atan2f(y, x);
    const bool big = mn > 0.414213562f * mx;
    const float t = (big ? mn - mx : mn) * __frcp_rn(big ? mn + mx : mx);
    const float z = t * t;
    // t - t z (1/3 - z/5 + z^2/7 - z^3/9 + z^4/11 - z^5/13 + z^6/15)
    const float p = fmaf(z, fmaf(z, fmaf(z, fmaf(z, fmaf(z, fmaf(z, 0.0666666667f, -0.0769230769f), 0.0909090909f),
                                              -0.111111111f), 0.142857143f), -0.2f), 0.333333333f);
    float th = fmaf(-t * z, p, t);
    if (big) th += 0.785398163f;
    if (ay > ax) th = 1.57079633f - th;
    if (x < 0.0f) th = 3.14159265f - th;
    return copysignf(th, y);
}

}  // namespace tro
