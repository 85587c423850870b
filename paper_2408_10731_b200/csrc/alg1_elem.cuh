// Per-element AM/AL update of Alg. 1 (solver_single.py:214-343), shared by the
// fused kernels.  Everything here is registers-only arithmetic on one
// (member, obstacle, sample) element.
#pragma once
#include "common.cuh"
#include "fastmath.cuh"

namespace tro {

// cos/sin of atan2(s, c) without trigonometry: (c, s) / hypot(c, s)
__device__ __forceinline__ void unit_dir(double c, double s, double* cu, double* su) {
    const double h2 = fma(c, c, s * s);
    if (h2 > 0.0) {
        const double r = rsqrt_fast(h2);
        *cu = c * r;
        *su = s * r;
    } else {  // atan2(+-0, +-0) = 0 or pi
        *cu = flip_sign(1.0, sign_bit(c));
        *su = flip_sign(0.0, sign_bit(s));
    }
}
__device__ __forceinline__ void unit_dir(float c, float s, float* cu, float* su) {
    const float h2 = fmaf(c, c, s * s);
    if (h2 > 0.0f) {
        const float r = rsqrt_fast(h2);
        *cu = c * r;
        *su = s * r;
    } else {
        *cu = signbit(c) ? -1.0f : 1.0f;
        *su = copysignf(0.0f, s);
    }
}

// d = min(max(1, sqrt(q)), 1e6) (solver_single.py:283-290) without fmin/fmax:
// q <= 1 <=> sqrt(q) <= 1 and q >= 1e12 <=> sqrt(q) >= 1e6 (sqrt is monotone, exact at both)
template <typename T>
__device__ __forceinline__ T los_scale(T q) {
    const T s = sqrt_fast(q > (T)1 ? q : (T)1);
    return q > (T)1e12 ? (T)1e6 : s;
}

template <typename T>
__device__ __forceinline__ T max_abs(T acc, T v) {
    v = fabs(v);
    return v > acc ? v : acc;
}
// running max of |x| kept as a SIGNED value: |.| is a free operand modifier of the compare, so one
// step is DSETP + 2 FSEL (max_abs materialises |v| first); the caller takes fabs of the result
template <typename T>
__device__ __forceinline__ T max_mag(T acc, T v) {
    return fabs(v) > fabs(acc) ? v : acc;
}

// Per-element words of the persistent state.
//   angle layout (LAY 0, the reference's variables):
//     3-D [alpha beta lx ly lz lca lsa lcb lsb] (9), 2-D [alpha lx ly lca lsa] (5)
//   unit layout (LAY 1): each angle is kept as its unit vector (cos, sin), which removes
//     the atan2 -> sincos round trip from every iteration at +2 (3-D) / +1 (2-D) words:
//     3-D [ca sa cb sb lx ly lz lca lsa lcb lsb] (11), 2-D [ca sa lx ly lca lsa] (6)
//   half layout (LAY 2): the reference's word count (9 / 5) with each angle stored as a folded
//     half-angle tangent (half_encode): cos / sin come back through one reciprocal and a few FMAs
//     (half_decode), so neither atan2 nor sin / cos runs per element and per iteration.
constexpr int kLayAngle = 0, kLayUnit = 1, kLayHalf = 2;
template <int DIM, int LAY>
struct Words {
    static constexpr int NA = DIM == 3 ? 2 : 1;          // angles
    static constexpr int NL = DIM == 3 ? 7 : 4;          // multiplier planes
    static constexpr int NV = LAY == kLayUnit ? 2 * NA : NA;  // words holding the angles
    static constexpr int W = NV + NL;
};

// Folded half-angle tangent of a unit vector (c, s) = (cos a, sin a):
//   c >= 0: w = tan(a / 2) = s / (1 + c) in [-1, 1];
//   c <  0: w = 3 sgn(s) + tan(b / 2) with b = a - pi sgn(s) (cos b = -c > 0): |w| in (2, 3].
// Both branches divide by a number >= 1, so the encoding never loses precision (tan(a / 2) alone
// blows up at a = pi).  Decoding is the rational parametrisation (1 - t^2, 2 t) / (1 + t^2).
template <typename T>
__device__ __forceinline__ T half_encode(T c, T s) {
    const bool pos = c >= (T)0;
    const T t = s * rcp_fast2ulp(pos ? (T)1 + c : (T)1 - c);
    return pos ? t : copysign((T)3, s) - t;
}
template <typename T>
__device__ __forceinline__ void half_decode(T w, T* c, T* s) {
    const bool inner = fabs(w) <= (T)1;
    const T t = inner ? w : w - copysign((T)3, w);
    const T t2 = t * t;
    const T q = rcp_fast2ulp((T)1 + t2);
    const T cc = ((T)1 - t2) * q, ss = (T)2 * t * q;
    *c = inner ? cc : -cc;
    *s = inner ? ss : -ss;
}

// Two reciprocals for the price of one (x, y >= 1 here, so x y neither overflows nor underflows):
// 1/x = y (1/(x y)), 1/y = x (1/(x y)), <= 2 ulp instead of <= 1 ulp each.  The element's independent
// pairs (the two angle decodes, the two encodes, the alpha- and beta-copy denominators) share one.
#ifndef TRO_RCP2
#define TRO_RCP2 1
#endif
template <typename T>
__device__ __forceinline__ void rcp2(T x, T y, T& rx, T& ry) {
#if TRO_RCP2
    const T r = rcp_fast2ulp(x * y);
    rx = y * r;
    ry = x * r;
#else
    rx = rcp_fast2ulp(x);
    ry = rcp_fast2ulp(y);
#endif
}
template <typename T>
__device__ __forceinline__ void half_decode2(T w1, T w2, T* c1, T* s1, T* c2, T* s2) {
    const bool in1 = fabs(w1) <= (T)1, in2 = fabs(w2) <= (T)1;
    const T t1 = in1 ? w1 : w1 - copysign((T)3, w1);
    const T t2 = in2 ? w2 : w2 - copysign((T)3, w2);
    const T u1 = t1 * t1, u2 = t2 * t2;
    T q1, q2;
    rcp2((T)1 + u1, (T)1 + u2, q1, q2);
    const T cc1 = ((T)1 - u1) * q1, ss1 = (T)2 * t1 * q1;
    const T cc2 = ((T)1 - u2) * q2, ss2 = (T)2 * t2 * q2;
    *c1 = in1 ? cc1 : -cc1;
    *s1 = in1 ? ss1 : -ss1;
    *c2 = in2 ? cc2 : -cc2;
    *s2 = in2 ? ss2 : -ss2;
}
template <typename T>
__device__ __forceinline__ void half_encode2(T c1, T s1, T c2, T s2, T* w1, T* w2) {
    const bool p1 = c1 >= (T)0, p2 = c2 >= (T)0;
    T r1, r2;
    rcp2(p1 ? (T)1 + c1 : (T)1 - c1, p2 ? (T)1 + c2 : (T)1 - c2, r1, r2);
    const T t1 = s1 * r1, t2 = s2 * r2;
    *w1 = p1 ? t1 : copysign((T)3, s1) - t1;
    *w2 = p2 ? t2 : copysign((T)3, s2) - t2;
}

// One AM iteration of one element.  v[W]: state words in / out.  (dx, dy, dz): the new position minus the
// obstacle centre.  d_old: the line-of-sight scale of the previous iterate.  Outputs the new d, the angle
// copies (for the optional export), the element's residual sum of squares `ss` and max-abs `ml`, and the
// target offsets off[] = target - obstacle centre the next position step sums (solver_single.py:177-189);
// the new position multipliers are v[o .. o + DIM).  The caller accumulates (in double, or in the storage
// type inside a thread for the fp32 build).
template <int DIM, typename T, int LAY>
__device__ __forceinline__ void am_element(T* v, T dx, T dy, T dz, T a, T b, T ia2, T ib2, T dold, T trho, T trho_o,
                                           T& ss_out, T& ml_out, T* off, T& dn, T* copies) {
    if constexpr (DIM == 3) {
        constexpr int o = LAY == kLayUnit ? 4 : 2;  // first multiplier word
        T sa, ca, sb, cb;
        if constexpr (LAY == kLayUnit) {
            ca = v[0]; sa = v[1]; cb = v[2]; sb = v[3];
        } else if constexpr (LAY == kLayHalf) {
            half_decode2(v[0], v[1], &ca, &sa, &cb, &sb);
        } else {
            sincos_fast(v[0], &sa, &ca);  // copy reset (solver_single.py:375-380)
            sincos_fast(v[1], &sb, &cb);
        }
        T lx = v[o], ly = v[o + 1], lz = v[o + 2], lca = v[o + 3], lsa = v[o + 4], lcb = v[o + 5], lsb = v[o + 6];
        // alpha copies (solver_single.py:223-228) and the beta-copy denominator (:253-266), one reciprocal
        const T coef = a * dold * sb;
        const T ccb = b * dold;
        T rden, rbden;
        rcp2(trho + trho_o * (coef * coef), trho + trho_o * (ccb * ccb), rden, rbden);
        const T Lx = lx + trho_o * dx, Ly = ly + trho_o * dy, Lz = lz + trho_o * dz;
        const T ca2 = (trho * ca - lca + coef * Lx) * rden;
        const T sa2 = (trho * sa - lsa + coef * Ly) * rden;
        // beta copies with the new alpha copies (solver_single.py:253-266)
        const T cb2 = (trho * cb - lcb + ccb * Lz) * rbden;
        const T csb = a * dold;
        const T num = trho * sb - lsb + csb * (ca2 * Lx + sa2 * Ly);
        const T sb2 = num * rcp_fast2ulp(trho + trho_o * (csb * csb) * (ca2 * ca2 + sa2 * sa2));
        // d from the new positions (solver_single.py:283-290)
        dn = los_scale(dx * dx * ia2 + dy * dy * ia2 + dz * dz * ib2);
        T cA2, sA2, cB2, sB2;
        unit_dir(ca2, sa2, &cA2, &sA2);  // cos/sin(alpha') for residuals + next targets
        unit_dir(cb2, sb2, &cB2, &sB2);
        if constexpr (LAY == kLayUnit) {
            v[0] = cA2; v[1] = sA2; v[2] = cB2; v[3] = sB2;
        } else if constexpr (LAY == kLayHalf) {
            half_encode2(cA2, sA2, cB2, sB2, &v[0], &v[1]);
        } else {
            v[0] = atan2_fast(sa2, ca2);  // solver_single.py:242
            v[1] = atan2_fast(sb2, cb2);  // solver_single.py:271
        }
        // residual families (solver_single.py:303-312)
        const T adn = a * dn;
        const T rx = dx - adn * ca2 * sb2;
        const T ry = dy - adn * sa2 * sb2;
        const T rz = dz - b * dn * cb2;
        const T rcb = cb2 - cB2, rsb = sb2 - sB2, rca = ca2 - cA2, rsa = sa2 - sA2;
        T ss = rx * rx;
        ss = fma(ry, ry, ss); ss = fma(rz, rz, ss); ss = fma(rcb, rcb, ss);
        ss = fma(rsb, rsb, ss); ss = fma(rca, rca, ss); ss = fma(rsa, rsa, ss);
        ss_out = ss;
        T ml = max_mag(rx, ry);
        ml = max_mag(ml, rz); ml = max_mag(ml, rcb);
        ml = max_mag(ml, rsb); ml = max_mag(ml, rca); ml = max_mag(ml, rsa);
        ml_out = fabs(ml);
        // multiplier ascent (solver_single.py:336-343)
        v[o] = lx + trho_o * rx; v[o + 1] = ly + trho_o * ry; v[o + 2] = lz + trho_o * rz;
        v[o + 3] = lca + trho * rca; v[o + 4] = lsa + trho * rsa;
        v[o + 5] = lcb + trho * rcb; v[o + 6] = lsb + trho * rsb;
        copies[0] = ca2; copies[1] = sa2; copies[2] = cb2; copies[3] = sb2;
        // the next position step's targets use the reset copies cos/sin of the new angles (solver_single.py:
        // 177-189, 204-207)
        off[0] = adn * cA2 * sB2;
        off[1] = adn * sA2 * sB2;
        off[2] = b * dn * cB2;
    } else {
        constexpr int o = LAY == kLayUnit ? 2 : 1;
        T sa, ca;
        if constexpr (LAY == kLayUnit) {
            ca = v[0]; sa = v[1];
        } else if constexpr (LAY == kLayHalf) {
            half_decode(v[0], &ca, &sa);
        } else {
            sincos_fast(v[0], &sa, &ca);
        }
        T lx = v[o], ly = v[o + 1], lca = v[o + 2], lsa = v[o + 3];
        // planar alpha copies (solver_single.py:229-237)
        const T cx = a * dold, cy = b * dold;
        const T ca2 = (trho * ca - lca + cx * (lx + trho_o * dx)) * rcp_fast(trho + trho_o * (cx * cx));
        const T sa2 = (trho * sa - lsa + cy * (ly + trho_o * dy)) * rcp_fast(trho + trho_o * (cy * cy));
        dn = los_scale(dx * dx * ia2 + dy * dy * ib2);
        T cA2, sA2;
        unit_dir(ca2, sa2, &cA2, &sA2);
        if constexpr (LAY == kLayUnit) {
            v[0] = cA2; v[1] = sA2;
        } else if constexpr (LAY == kLayHalf) {
            v[0] = half_encode(cA2, sA2);
        } else {
            v[0] = atan2_fast(sa2, ca2);
        }
        const T rx = dx - a * dn * ca2;
        const T ry = dy - b * dn * sa2;
        const T rca = ca2 - cA2, rsa = sa2 - sA2;
        T ss = rx * rx;
        ss = fma(ry, ry, ss); ss = fma(rca, rca, ss); ss = fma(rsa, rsa, ss);
        ss_out = ss;
        T ml = max_mag(rx, ry);
        ml = max_mag(ml, rca); ml = max_mag(ml, rsa);
        ml_out = fabs(ml);
        v[o] = lx + trho_o * rx; v[o + 1] = ly + trho_o * ry;
        v[o + 2] = lca + trho * rca; v[o + 3] = lsa + trho * rsa;
        copies[0] = ca2; copies[1] = sa2;
        off[0] = a * dn * cA2;
        off[1] = b * dn * sA2;
    }
}

// Cold-start angles / prime of a state (no update): fills v for INIT, then the
// residual of the copies-reset state (copies == cos/sin of the angles, so only the
// collision families are non-zero) and the sums the first position step needs.
template <int DIM, typename T, int LAY, bool INIT>
__device__ __forceinline__ void prime_element(T* v, double trx, double trY, double trz, double px, double py,
                                              double pz, double ad, double bd, T dold, double& sumsq, double& mx,
                                              double* accL, double* accT) {
    constexpr int NL = Words<DIM, LAY>::NL;
    constexpr int o = Words<DIM, LAY>::NV;
    const double ex = px - trx, ey = py - trY, ez = pz - trz;
    T ca, sa, cb = 0, sb = 0;
    if constexpr (INIT) {
        // angles of the straight-line offsets: angles3d (geometry.py:102-114) in 3-D, the
        // ellipse-scaled angle2d in 2-D (solver_single.py:138-143); -pi folds onto pi
        double a0 = DIM == 3 ? atan2(ey, ex) : atan2(ey / bd, ex / ad);
        if (a0 == -M_PI) a0 = M_PI;
        double b0 = DIM == 3 ? atan2(hypot(ex / ad, ey / ad), ez / bd) : 0.0;
        double s0, c0, s1, c1;
        sincos(a0, &s0, &c0);
        sincos(b0, &s1, &c1);
        if constexpr (LAY == kLayUnit) {
            v[0] = (T)c0; v[1] = (T)s0;
            if (DIM == 3) { v[2] = (T)c1; v[3] = (T)s1; }
        } else if constexpr (LAY == kLayHalf) {
            v[0] = half_encode((T)c0, (T)s0);
            if (DIM == 3) v[1] = half_encode((T)c1, (T)s1);
        } else {
            v[0] = (T)a0;
            if (DIM == 3) v[1] = (T)b0;
        }
#pragma unroll
        for (int k = 0; k < NL; ++k) v[o + k] = (T)0;
    }
    if constexpr (LAY == kLayUnit) {
        ca = v[0]; sa = v[1];
        if (DIM == 3) { cb = v[2]; sb = v[3]; }
    } else if constexpr (LAY == kLayHalf) {
        half_decode(v[0], &ca, &sa);
        if (DIM == 3) half_decode(v[1], &cb, &sb);
    } else {
        sincos_fast(v[0], &sa, &ca);
        if (DIM == 3) sincos_fast(v[1], &sb, &cb);
    }
    const T a = (T)ad, b = (T)bd;
    double rr, ml;
    if constexpr (DIM == 3) {
        const T rx = (T)ex - a * dold * ca * sb, ry = (T)ey - a * dold * sa * sb, rz = (T)ez - b * dold * cb;
        rr = (double)rx * rx + (double)ry * ry + (double)rz * rz;
        ml = fmax(fmax(fabs((double)rx), fabs((double)ry)), fabs((double)rz));
        accT[0] += trx + (double)(a * dold * ca * sb);
        accT[1] += trY + (double)(a * dold * sa * sb);
        accT[2] += trz + (double)(b * dold * cb);
    } else {
        const T rx = (T)ex - a * dold * ca, ry = (T)ey - b * dold * sa;
        rr = (double)rx * rx + (double)ry * ry;
        ml = fmax(fabs((double)rx), fabs((double)ry));
        accT[0] += trx + (double)(a * dold * ca);
        accT[1] += trY + (double)(b * dold * sa);
    }
    sumsq += rr;
    mx = ml > mx ? ml : mx;
#pragma unroll
    for (int ax = 0; ax < DIM; ++ax) accL[ax] += (double)v[o + ax];
}

}  // namespace tro
