// dd.cuh — double-double (FP64-pair) arithmetic for the leaf, frontier and reduction kernels.
//
// A dd value is hi + lo with |lo| <= ulp(hi)/2.  Error-free transforms: TwoSum (Knuth) and the
// FMA product error.  Products drop the lo*lo term (relative error <= ~2^-104).  Used because the
// combination sum is ill-conditioned (Eq 2.8 negative weights):
// per-point FP64 cannot meet 1e-12 on configs 4-5, dd partial products can.
#pragma once
#include <cuda_runtime.h>
#include <math.h>

#define DD_HD __host__ __device__ __forceinline__

struct dd {
    double hi, lo;
};
struct cdd {   // complex dd (oscillatory kind): re + i im
    dd re, im;
};

DD_HD dd dd_make(double h, double l = 0.0) { return dd{h, l}; }

DD_HD void two_sum(double a, double b, double &s, double &e) {
    s = a + b;
    double bb = s - a;
    e = (a - (s - bb)) + (b - bb);
}
DD_HD void quick_two_sum(double a, double b, double &s, double &e) {
    s = a + b;
    e = b - (s - a);
}
DD_HD dd dd_norm(double p, double e) {
    dd r;
    quick_two_sum(p, e, r.hi, r.lo);
    return r;
}
// accurate dd + dd
DD_HD dd dd_add(dd a, dd b) {
    double s, e, t, f;
    two_sum(a.hi, b.hi, s, e);
    two_sum(a.lo, b.lo, t, f);
    e += t;
    quick_two_sum(s, e, s, e);
    e += f;
    dd r;
    quick_two_sum(s, e, r.hi, r.lo);
    return r;
}
DD_HD dd dd_neg(dd a) { return dd{-a.hi, -a.lo}; }
DD_HD dd dd_sub(dd a, dd b) { return dd_add(a, dd_neg(b)); }
// unnormalised product: a*b = p + e (lo*lo dropped)
DD_HD void dd_mul_pe(dd a, dd b, double &p, double &e) {
    p = a.hi * b.hi;
    e = fma(a.hi, b.hi, -p);
    e = fma(a.hi, b.lo, e);
    e = fma(a.lo, b.hi, e);
}
DD_HD dd dd_mul(dd a, dd b) {
    double p, e;
    dd_mul_pe(a, b, p, e);
    return dd_norm(p, e);
}
DD_HD dd dd_mul_d(dd a, double b) {
    double p = a.hi * b;
    double e = fma(a.hi, b, -p);
    e = fma(a.lo, b, e);
    return dd_norm(p, e);
}
DD_HD dd dd_from_prod(double a, double b) {   // exact product of two doubles
    double p = a * b;
    return dd{p, fma(a, b, -p)};
}
DD_HD dd dd_from_sum(double a, double b) {    // exact sum of two doubles
    dd r;
    two_sum(a, b, r.hi, r.lo);
    return r;
}
DD_HD dd dd_div(dd a, dd b) {
    double q1 = a.hi / b.hi;
    dd r = dd_sub(a, dd_mul_d(b, q1));
    double q2 = r.hi / b.hi;
    r = dd_sub(r, dd_mul_d(b, q2));
    double q3 = r.hi / b.hi;
    dd q = dd_norm(q1, q2);
    return dd_add(q, dd{q3, 0.0});
}
DD_HD dd dd_div_d(dd a, double b) { return dd_div(a, dd{b, 0.0}); }
// 1 / y: FP64 quotient r0 and one Newton correction r0 (1 + e), e = 1 - y r0 (two FMAs): ~2^-104
DD_HD dd dd_recip(dd y) {
    const double r0 = 1.0 / y.hi;
    double e = fma(-y.hi, r0, 1.0);
    e = fma(-y.lo, r0, e);
    return dd_norm(r0, r0 * e);
}
DD_HD cdd cdd_mul(cdd a, cdd b) {
    cdd r;
    r.re = dd_sub(dd_mul(a.re, b.re), dd_mul(a.im, b.im));
    r.im = dd_add(dd_mul(a.re, b.im), dd_mul(a.im, b.re));
    return r;
}
DD_HD cdd cdd_mul_dd(cdd a, dd b) { return cdd{dd_mul(a.re, b), dd_mul(a.im, b)}; }

// "sloppy" dd addition (one TwoSum on the high parts, low parts added in FP64): 11 FP64 ops instead
// of 20; error <= ~2^-104 (|a| + |b|), which is all the leaf partial sums need (their own grid error
// is relative to the same bound).
DD_HD dd dd_add_fast(dd a, dd b) {
    double s, e;
    two_sum(a.hi, b.hi, s, e);
    e += a.lo + b.lo;
    return dd_norm(s, e);
}
// x +/- y for two unnormalised products (p, e) = dd_mul_pe outputs, renormalised: 11 FP64 ops
DD_HD dd dd_combine_pe(double px, double ex, double py, double ey) {
    double s, e;
    two_sum(px, py, s, e);
    e += ex + ey;
    return dd_norm(s, e);
}
// complex dd product from four shared unnormalised products: 4 x (1 DMUL + 3 DFMA) + 2 x 11
DD_HD cdd cdd_mul_fast(cdd a, cdd b) {
    double p1, e1, p2, e2, p3, e3, p4, e4;
    dd_mul_pe(a.re, b.re, p1, e1);
    dd_mul_pe(a.im, b.im, p2, e2);
    dd_mul_pe(a.re, b.im, p3, e3);
    dd_mul_pe(a.im, b.re, p4, e4);
    return cdd{dd_combine_pe(p1, e1, -p2, -e2), dd_combine_pe(p3, e3, p4, e4)};
}
// a * b and a * conj(b) sharing the four products (symmetric node pairs: F_0 = conj(F_2))
DD_HD void cdd_mul_conj_pair(cdd a, cdd b, cdd &ab, cdd &abc) {
    double p1, e1, p2, e2, p3, e3, p4, e4;
    dd_mul_pe(a.re, b.re, p1, e1);
    dd_mul_pe(a.im, b.im, p2, e2);
    dd_mul_pe(a.re, b.im, p3, e3);
    dd_mul_pe(a.im, b.re, p4, e4);
    ab = cdd{dd_combine_pe(p1, e1, -p2, -e2), dd_combine_pe(p3, e3, p4, e4)};
    abc = cdd{dd_combine_pe(p1, e1, p2, e2), dd_combine_pe(p4, e4, -p3, -e3)};
}

// ---------------------------------------------------------------------------------------------
// Transcendentals in dd (plan-time factor tables, K0).  Accuracy ~1e-31 relative on the ranges used
// (|x| < 700 for exp; any |x| for sin/cos via reduction with a 3-part 2*pi).
// ---------------------------------------------------------------------------------------------
#define DD_LN2_HI 6.931471805599453e-01
#define DD_LN2_LO 2.3190468138462996e-17
// 2*pi as three doubles (hi + mid + lo)
#define DD_2PI_0 6.283185307179586e+00
#define DD_2PI_1 2.4492935982947064e-16
#define DD_2PI_2 -5.989539619436679e-33
#define DD_PI2_HI 1.5707963267948966e+00
#define DD_PI2_LO 6.123233995736766e-17
#define DD_PI2_LO2 -1.4973849048591698e-33

DD_HD dd dd_ldexp(dd a, int e) { return dd{ldexp(a.hi, e), ldexp(a.lo, e)}; }

#ifdef __CUDACC__
// Reciprocal constants for the Taylor series below (dd, from 60-digit values): multiplying by
// them replaces the dd divisions of the Horner steps.
// 1/n, n = 0..14 (index n), as dd (hi, lo)
__device__ __constant__ double DD_INV_N[15][2] = {
    {0.0, 0.0},
    {1.0, 0.0},
    {0.5, 0.0},
    {0.3333333333333333, 1.850371707708594e-17},
    {0.25, 0.0},
    {0.2, -1.1102230246251566e-17},
    {0.16666666666666666, 9.25185853854297e-18},
    {0.14285714285714285, 7.93016446160826e-18},
    {0.125, 0.0},
    {0.1111111111111111, 6.1679056923619804e-18},
    {0.1, -5.551115123125783e-18},
    {0.09090909090909091, -2.523234146875356e-18},
    {0.08333333333333333, 4.625929269271485e-18},
    {0.07692307692307693, -4.270088556250602e-18},
    {0.07142857142857142, 3.96508223080413e-18}
};
// 1/((2n)(2n+1)) and 1/((2n-1)(2n)), n = 0..13
__device__ __constant__ double DD_INV_SIN[14][2] = {
    {0.0, 0.0},
    {0.16666666666666666, 9.25185853854297e-18},
    {0.05, -2.7755575615628915e-18},
    {0.023809523809523808, 1.32169407693471e-18},
    {0.013888888888888888, 7.709882115452476e-19},
    {0.00909090909090909, 4.415659757031872e-19},
    {0.00641025641025641, 2.2240044563805217e-19},
    {0.004761904761904762, -4.295505750037808e-19},
    {0.003676470588235294, 5.102127870520021e-20},
    {0.0029239766081871343, 1.6231330769373633e-19},
    {0.002380952380952381, -2.147752875018904e-19},
    {0.001976284584980237, 1.3370398332627564e-19},
    {0.0016666666666666668, -1.0697461435190311e-19},
    {0.0014245014245014246, -7.104458680104445e-20}
};
__device__ __constant__ double DD_INV_COS[14][2] = {
    {0.0, 0.0},
    {0.5, 0.0},
    {0.08333333333333333, 4.625929269271485e-18},
    {0.03333333333333333, 4.625929269271486e-19},
    {0.017857142857142856, 9.912705577010326e-19},
    {0.011111111111111112, -4.2404351634988616e-19},
    {0.007575757575757576, -2.1026951223961299e-19},
    {0.005494505494505495, -4.2891514515910067e-19},
    {0.004166666666666667, 5.782411586589357e-20},
    {0.0032679738562091504, -9.920804192677818e-20},
    {0.002631578947368421, 5.934580312552235e-20},
    {0.0021645021645021645, 1.8774063592822588e-21},
    {0.0018115942028985507, -2.199830494898125e-20},
    {0.0015384615384615385, 1.3344026738283131e-21}
};

#define DD_DEV __device__ __forceinline__


// exp(a): a = m ln2 + r, r /= 2^6, Taylor to r^14 (|r| < 5.5e-3 -> truncation < 1e-45),
// then 6 squarings in expm1 form t <- 2t + t^2 (error growth x64), result (1 + t) 2^m.
DD_DEV dd dd_exp(dd a) {
    if (a.hi == 0.0 && a.lo == 0.0) return dd{1.0, 0.0};
    double m = rint(a.hi / DD_LN2_HI);
    dd r = dd_sub(a, dd_add(dd_from_prod(m, DD_LN2_HI), dd_from_prod(m, DD_LN2_LO)));
    r = dd_ldexp(r, -6);
    // expm1(r) = r + r^2/2! + ... + r^14/14!  (Horner: r(1 + r/2(1 + r/3(...))))
    dd t = dd{1.0, 0.0};
    for (int n = 14; n >= 2; --n)
        t = dd_add(dd{1.0, 0.0}, dd_mul(dd_mul(r, t), dd{DD_INV_N[n][0], DD_INV_N[n][1]}));
    t = dd_mul(r, t);
    for (int i = 0; i < 6; ++i) t = dd_add(dd_ldexp(t, 1), dd_mul(t, t));
    dd e = dd_add(dd{1.0, 0.0}, t);
    return dd_ldexp(e, (int)m);
}

// sin and cos of r with |r| <= pi/4 by Taylor series (terms to r^27: truncation < 1e-34).
DD_DEV void dd_sincos_small(dd r, dd &s, dd &c) {
    dd r2 = dd_mul(r, r);
    // sin = r (1 - r2/(2*3) (1 - r2/(4*5) (1 - ...)))
    dd ts = dd{1.0, 0.0}, tc = dd{1.0, 0.0};
    for (int n = 13; n >= 1; --n) {
        ts = dd_sub(dd{1.0, 0.0}, dd_mul(dd_mul(r2, ts), dd{DD_INV_SIN[n][0], DD_INV_SIN[n][1]}));
        tc = dd_sub(dd{1.0, 0.0}, dd_mul(dd_mul(r2, tc), dd{DD_INV_COS[n][0], DD_INV_COS[n][1]}));
    }
    s = dd_mul(r, ts);
    c = tc;
}

// sin/cos of a dd argument: reduce by 2*pi (3-part), then by pi/2 to |r| <= pi/4.
DD_DEV void dd_sincos(dd a, dd &s, dd &c) {
    double n2 = rint(a.hi / DD_2PI_0);
    dd x = a;
    if (n2 != 0.0) {
        x = dd_sub(x, dd_from_prod(n2, DD_2PI_0));
        x = dd_sub(x, dd_from_prod(n2, DD_2PI_1));
        x = dd_sub(x, dd{n2 * DD_2PI_2, 0.0});
    }
    double q = rint(x.hi / DD_PI2_HI);
    int qi = (int)q;
    if (q != 0.0) {
        x = dd_sub(x, dd_from_prod(q, DD_PI2_HI));
        x = dd_sub(x, dd_from_prod(q, DD_PI2_LO));
        x = dd_sub(x, dd{q * DD_PI2_LO2, 0.0});
    }
    dd ss, cc;
    dd_sincos_small(x, ss, cc);
    switch (((qi % 4) + 4) % 4) {
    case 0: s = ss; c = cc; break;
    case 1: s = cc; c = dd_neg(ss); break;
    case 2: s = dd_neg(ss); c = dd_neg(cc); break;
    default: s = dd_neg(cc); c = ss; break;
    }
}
#endif  // __CUDACC__

// Out-of-line copies for the latency-bound K0 / head launches: one body per kernel however many call
// sites (the factor entry and the base), so the cold launch fetches less code.
__device__ __noinline__ dd dd_exp_ool(dd a) { return dd_exp(a); }
__device__ __noinline__ void dd_sincos_ool(dd a, dd &s, dd &c) { dd_sincos(a, s, c); }
__device__ __noinline__ dd dd_div_ool(dd a, dd b) { return dd_div(a, b); }
