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
// Constants of the table-driven exp / sin / cos below (60-digit values split into dd hi + lo;
// generated by tools/gen_dd_consts.py).
// 1/(k+1)!, k = 0..11 (exp(s) - 1 = s sum_k s^k/(k+1)!)
__device__ __constant__ double DD_EXP_C[12][2] = {
    {1.0, 0.0},
    {0.5, 0.0},
    {0.16666666666666666, 9.25185853854297e-18},
    {0.041666666666666664, 2.3129646346357427e-18},
    {0.008333333333333333, 1.1564823173178714e-19},
    {0.001388888888888889, -5.300543954373577e-20},
    {0.0001984126984126984, 1.7209558293420705e-22},
    {2.48015873015873e-05, 2.1511947866775882e-23},
    {2.7557319223985893e-06, -1.858393274046472e-22},
    {2.755731922398589e-07, 2.3767714622250297e-23},
    {2.505210838544172e-08, -1.448814070935912e-24},
    {2.08767569878681e-09, -1.20734505911326e-25}
};
// exp(j/64), j = -23..23 (index j + 23)
__device__ __constant__ double DD_EXP_TAB[47][2] = {
    {0.6981125100681258, 4.379112262891346e-17},
    {0.7091061824373984, -1.2868055655346304e-17},
    {0.7202729799554398, -3.7374088280484695e-17},
    {0.7316156289466418, 8.35576468031604e-18},
    {0.7431368986687583, -9.001102395673582e-19},
    {0.7548396019890073, -9.844076038651084e-18},
    {0.76672659607082, 2.5682592802096574e-17},
    {0.7788007830714049, -1.0231869534531498e-17},
    {0.791065110850296, 5.426586044764942e-17},
    {0.8035225736890608, -3.661886830920417e-17},
    {0.8161762130223398, 6.554697808700811e-18},
    {0.8290291181804004, -2.7604408719539223e-17},
    {0.8420844271433824, -3.8967887440685524e-17},
    {0.8553453273074225, 1.7204900005057594e-17},
    {0.8688150562628432, 6.146598011714697e-19},
    {0.8824969025845955, -5.224526916735663e-17},
    {0.8963942066351505, -4.7460497709066285e-17},
    {0.9105103613800342, -3.325048324577564e-17},
    {0.9248488132162048, 1.0614261758612887e-17},
    {0.9394130628134758, -2.152447043447057e-17},
    {0.9542066659691884, -3.392457164103672e-17},
    {0.9692332344763441, -4.801151707083219e-17},
    {0.9844964370054085, -4.7493026566356186e-17},
    {1.0, 0.0},
    {1.0157477085866857, 2.0530467874932267e-17},
    {1.0317434074991028, -8.944417741043132e-17},
    {1.0479910020166328, -5.327900898877614e-17},
    {1.0644944589178593, 1.0872888143211957e-16},
    {1.0812578074490395, 6.013904942011385e-17},
    {1.0982851403078258, 9.070644949793751e-17},
    {1.1155806146424807, 5.298211318168963e-17},
    {1.1331484530668263, -5.370737708558031e-18},
    {1.1509929446911764, 3.7613173622701076e-17},
    {1.1691184461695043, 6.945488167320411e-17},
    {1.1875293827631006, 6.415816207759217e-19},
    {1.2062302494209807, 3.9295715071105525e-17},
    {1.2252256118773075, 8.279379001181868e-17},
    {1.2445201077660952, -7.440512295261056e-17},
    {1.2641184477534664, -1.541497933603795e-17},
    {1.2840254166877414, 8.968972781793724e-17},
    {1.3042458747676378, 1.7093578107981658e-17},
    {1.3247847587288655, 9.422682377542367e-17},
    {1.3456470830494105, 3.415854209639032e-17},
    {1.3668379411737963, 5.1449446596411544e-17},
    {1.3883625067566268, 6.691963657219203e-17},
    {1.4102260349257107, -4.1758810273684196e-17},
    {1.4324338635650782, -6.53862212642198e-17}
};
// (-1)^k/(2k+1)!, k = 0..7
__device__ __constant__ double DD_SIN_C[8][2] = {
    {1.0, 0.0},
    {-0.16666666666666666, -9.25185853854297e-18},
    {0.008333333333333333, 1.1564823173178714e-19},
    {-0.0001984126984126984, -1.7209558293420705e-22},
    {2.7557319223985893e-06, -1.858393274046472e-22},
    {-2.505210838544172e-08, 1.448814070935912e-24},
    {1.6059043836821613e-10, 1.2585294588752098e-26},
    {-7.647163731819816e-13, -7.03872877733453e-30}
};
// (-1)^k/(2k)!, k = 0..7
__device__ __constant__ double DD_COS_C[8][2] = {
    {1.0, 0.0},
    {-0.5, 0.0},
    {0.041666666666666664, 2.3129646346357427e-18},
    {-0.001388888888888889, 5.300543954373577e-20},
    {2.48015873015873e-05, 2.1511947866775882e-23},
    {-2.755731922398589e-07, -2.3767714622250297e-23},
    {2.08767569878681e-09, -1.20734505911326e-25},
    {-1.1470745597729725e-11, -2.0655512752830745e-28}
};
// sin(j pi/64), j = 0..16
__device__ __constant__ double DD_SINPI64[17][2] = {
    {0.0, 0.0},
    {0.049067674327418015, -6.79610372051828e-19},
    {0.0980171403295606, -1.634582362244256e-18},
    {0.14673047445536175, 3.726947147046568e-18},
    {0.19509032201612828, -7.991079068461731e-18},
    {0.2429801799032639, -8.751431529719663e-18},
    {0.2902846772544624, -1.892797870777425e-17},
    {0.33688985339222005, -4.200094003347509e-19},
    {0.3826834323650898, -1.0050772696461588e-17},
    {0.4275550934302821, 9.411189816295473e-18},
    {0.47139673682599764, 6.516678136069013e-18},
    {0.5141027441932218, -4.5712707523615624e-17},
    {0.5555702330196022, 4.709410940561677e-17},
    {0.5956993044924334, -1.3438641936579467e-17},
    {0.6343932841636455, 1.0420901929280035e-17},
    {0.6715589548470184, -4.048903774929669e-17},
    {0.7071067811865476, -4.833646656726457e-17}
};
// cos(j pi/64), j = 0..16
__device__ __constant__ double DD_COSPI64[17][2] = {
    {1.0, 0.0},
    {0.9987954562051724, -1.2291693337075465e-17},
    {0.9951847266721969, -4.248691367830441e-17},
    {0.989176509964781, -4.098730993704711e-17},
    {0.9807852804032304, 1.8546939997825006e-17},
    {0.970031253194544, 1.8365300348428844e-17},
    {0.9569403357322088, 4.05538698618757e-17},
    {0.9415440651830208, -2.789637954769834e-17},
    {0.9238795325112867, 1.7645047084336677e-17},
    {0.9039892931234433, -6.609754468748431e-18},
    {0.881921264348355, -1.9843248405890562e-17},
    {0.8577286100002721, -4.818344793633662e-17},
    {0.8314696123025452, 1.4073856984728024e-18},
    {0.8032075314806449, -3.306060980481491e-17},
    {0.773010453362737, -3.256590703364977e-17},
    {0.7409511253549591, -1.4708616952297345e-17},
    {0.7071067811865476, -4.833646656726457e-17}
};
#define DD_PI64_0 0.04908738521234052
#define DD_PI64_1 1.9135106236677394e-18
#define DD_PI64_2 -4.6793278276849057e-35
#define DD_64_PI 20.371832715762604
#define DD_INV_LN2 1.4426950408889634

#define DD_DEV __device__ __forceinline__
#define DD_C(T, k) (dd{T[k][0], T[k][1]})

// The transcendentals are latency-bound (one dependent chain per thread in the K0 / head launches):
// table reduction to a short interval, then a short polynomial evaluated Estrin-style (independent
// dd products side by side instead of one long Horner chain), the tail coefficients whose terms are
// below 2^-60 of the result in plain FP64.  Critical path ~10 dd operations instead of ~40-55 for
// the Taylor-Horner forms they replace.

// exp(a) = 2^m exp(j/64) exp(s): a = m ln2 + j/64 + s, |s| <= 1/128 + tiny;
// exp(s) - 1 = s P(s), P(s) = sum_{k=0}^{11} s^k/(k+1)! (next term s^13/13! < 1e-37).
DD_DEV dd dd_exp(dd a) {
    if (a.hi == 0.0 && a.lo == 0.0) return dd{1.0, 0.0};
    const double m = rint(a.hi * DD_INV_LN2);
    const dd r = dd_sub(a, dd_add(dd_from_prod(m, DD_LN2_HI), dd_from_prod(m, DD_LN2_LO)));
    const double jd = fmin(fmax(rint(r.hi * 64.0), -23.0), 23.0);
    const dd x = dd_add(r, dd{-jd * 0.015625, 0.0});
    const double xh = x.hi;
    // k >= 7 in FP64 (those terms are < 5e-20 of P)
    const double h = DD_EXP_C[7][0] + xh * (DD_EXP_C[8][0] + xh * (DD_EXP_C[9][0] +
                                                               xh * (DD_EXP_C[10][0] + xh * DD_EXP_C[11][0])));
    const dd x2 = dd_mul(x, x);
    const dd e0 = dd_add(dd{1.0, 0.0}, dd_ldexp(x, -1));                     // 1 + x/2 (exact halving)
    const dd e1 = dd_add(DD_C(DD_EXP_C, 2), dd_mul(DD_C(DD_EXP_C, 3), x));
    const dd e2 = dd_add(DD_C(DD_EXP_C, 4), dd_mul(DD_C(DD_EXP_C, 5), x));
    const dd e3 = dd_add(DD_C(DD_EXP_C, 6), dd{xh * h, 0.0});
    const dd x4 = dd_mul(x2, x2);
    const dd f0 = dd_add(e0, dd_mul(x2, e1));
    const dd f1 = dd_add(e2, dd_mul(x2, e3));
    const dd P = dd_add(f0, dd_mul(x4, f1));
    const dd T = DD_C(DD_EXP_TAB, (int)jd + 23);
    const dd e = dd_add(T, dd_mul(T, dd_mul(x, P)));                        // T (1 + (e^x - 1))
    return dd_ldexp(e, (int)m);
}

// sin and cos of a dd argument: a = N pi/64 + t (one reduction, 3-part pi/64: |t| <= pi/128 + tiny),
// N = 32 Q + J with J in [-16, 15]; sin t = t S(t^2), cos t = C(t^2) (terms to t^15 / t^14:
// truncation < 1e-34); the angle sum with the dd table of J pi/64, then the quadrant Q mod 4.
DD_DEV void dd_sincos(dd a, dd &s, dd &c) {
    const double nd = rint(a.hi * DD_64_PI);
    dd t = a;
    if (nd != 0.0) {
        const dd K = dd_add(dd_from_prod(nd, DD_PI64_0), dd_from_prod(nd, DD_PI64_1));
        t = dd_add(dd_sub(a, K), dd{-nd * DD_PI64_2, 0.0});
    }
    const long long N = (long long)nd;
    const long long Q = (N + 16) >> 5;   // floor((N + 16) / 32)
    const int J = (int)(N - 32 * Q);     // -16 .. 15
    const dd u = dd_mul(t, t);
    const double uh = u.hi;
    // k >= 4 in FP64 (those terms are < 4e-19 of S, C)
    const double hs = DD_SIN_C[4][0] + uh * (DD_SIN_C[5][0] + uh * (DD_SIN_C[6][0] + uh * DD_SIN_C[7][0]));
    const double hc = DD_COS_C[4][0] + uh * (DD_COS_C[5][0] + uh * (DD_COS_C[6][0] + uh * DD_COS_C[7][0]));
    const dd u2 = dd_mul(u, u);
    const dd s0 = dd_add(dd{1.0, 0.0}, dd_mul(DD_C(DD_SIN_C, 1), u));
    const dd s1 = dd_add(DD_C(DD_SIN_C, 2), dd_mul(DD_C(DD_SIN_C, 3), u));
    const dd c0 = dd_add(dd{1.0, 0.0}, dd_neg(dd_ldexp(u, -1)));   // 1 - u/2 (exact halving)
    const dd c1 = dd_add(DD_C(DD_COS_C, 2), dd_mul(DD_C(DD_COS_C, 3), u));
    const dd gs = dd_add(s1, dd{u2.hi * hs, 0.0});
    const dd gc = dd_add(c1, dd{u2.hi * hc, 0.0});
    const dd st = dd_mul(t, dd_add(s0, dd_mul(u2, gs)));
    const dd ct = dd_add(c0, dd_mul(u2, gc));
    dd ss = st, cc = ct;
    if (J != 0) {
        const int ja = J < 0 ? -J : J;
        dd sj = DD_C(DD_SINPI64, ja);
        const dd cj = DD_C(DD_COSPI64, ja);
        if (J < 0) sj = dd_neg(sj);
        ss = dd_add(dd_mul(sj, ct), dd_mul(cj, st));
        cc = dd_sub(dd_mul(cj, ct), dd_mul(sj, st));
    }
    switch ((int)(Q & 3)) {
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
