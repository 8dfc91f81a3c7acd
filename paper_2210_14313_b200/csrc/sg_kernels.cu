// sg_kernels.cu — sm_100a kernels and the C ABI of the B200 Smolyak hot path.
//
//  K0  k_factor / k_base : per-(coordinate, level, node) factor table F = w * E_k(x) and the base B
//                          in double-double, on the device.  The integrand
//                          f(x) = Re(B * prod_{active k} E_k(x_k)) for all four kinds.
//  K2+K3 k_root / k_pass : level-synchronous prefix-tree passes (Eqs 3.8-3.11:
//                          the "multilevel dimension iteration").  Pass t reads frontier t (the
//                          extendable depth-t prefixes, each carrying its dd partial product
//                          P = B * prod w E), evaluates every depth-(t+1) Smolyak point
//                          term = coef[e] * Re(P * F[k'][l'][j']) and writes the extendable
//                          children into frontier t+1.
//  K4  block/grid reduce : fixed-order dd warp-shuffle butterfly -> CTA -> per-CTA partials ->
//                          single-CTA fixed-order pass (deterministic, bitwise reproducible).
#include <cuda_runtime.h>
#include <stdint.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

#include <algorithm>
#include <climits>
#include <new>
#include <vector>

#include "../../include/sg_b200.h"
#include "dd.cuh"
#include "plan.h"

#define WPB 8                 // warps per CTA in the pass kernels
#define PASS_THREADS (WPB * 32)
#define META_KMASK ((1u << SG_META_KBITS) - 1u)

struct DevPlan {
    int d, L, kind, nfront;
    int nl[SG_MAX_L + 3];
    int entry_off[SG_MAX_L + 3];
    int tab_off[SG_MAX_L + 3];
    double coef[SG_MAX_L + 2];
    long long M0;
    const double *X, *Whi, *Wlo;
    const double *c, *w, *u;
    double2 *Fre, *Fim;
    double *base;   // re.hi, re.lo, im.hi, im.lo
    double *SA;     // [(L+2) x (d+1)] suffix sums of |F| per level (k_leaf's accumulation bound)
    int *status;
    int sform;      // 0 factor form; 1 SG_ARITH_SFORM_FP64, 2 SG_ARITH_SFORM_DD: base[0..1] = argument S
    int symmask;    // bit l: level-l row symmetric about 1/2 (x_j = 1 - x_{n-1-j}, equal dd weights,
                    // the midpoint at the centre if n is odd): oscillatory factors of a pair are
                    // exact conjugates, the midpoint's is real (k_leaf's symmetric-row path)
    const double2 *coefm;   // node coefficient (dd) per (depth t, excess b): [t * (L + 1) + b]
};

struct PassArgs {
    long long nsrc, ntasks;
    int nsplit;
    int t;                         // depth of the source frontier (children have depth t + 1)
    const double2 *src_re, *src_im;
    const uint32_t *src_meta;
    double2 *dst_re, *dst_im;
    uint32_t *dst_meta;
    const long long *offT, *NT, *CT, *TB;
    double2 *partials;
    unsigned long long *counter;   // dynamic task counter (persistent kernels), zeroed per launch
};

struct RootArgs {
    long long lo, hi;
    const long long *off1, *JS;
    double2 *dst_re, *dst_im;
    uint32_t *dst_meta;
    double2 *partials;
};

// ---------------------------------------------------------------------------------------------
// reductions (K4)
// ---------------------------------------------------------------------------------------------
__device__ __forceinline__ dd warp_reduce_dd(dd v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
        dd w;
        w.hi = __shfl_xor_sync(0xffffffffu, v.hi, o);
        w.lo = __shfl_xor_sync(0xffffffffu, v.lo, o);
        v = dd_add(v, w);
    }
    return v;
}

// same butterfly with the sloppy dd add (leaf task partials; fixed order, deterministic)
__device__ __forceinline__ dd warp_reduce_dd_fast(dd v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
        dd w;
        w.hi = __shfl_xor_sync(0xffffffffu, v.hi, o);
        w.lo = __shfl_xor_sync(0xffffffffu, v.lo, o);
        v = dd_add_fast(v, w);
    }
    return v;
}

// CTA sum in fixed order; result valid in thread 0.
template <int NWARPS>
__device__ __forceinline__ dd block_reduce_dd(dd v) {
    __shared__ double2 sm[NWARPS];
    v = warp_reduce_dd(v);
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    if (lane == 0) sm[wid] = make_double2(v.hi, v.lo);
    __syncthreads();
    dd s = {0.0, 0.0};
    if (threadIdx.x == 0) {
        for (int i = 0; i < NWARPS; ++i) s = dd_add(s, dd{sm[i].x, sm[i].y});
    }
    return s;
}

// ---------------------------------------------------------------------------------------------
// K0: factor table and base
// ---------------------------------------------------------------------------------------------
__device__ __forceinline__ bool dd_finite(dd a) { return isfinite(a.hi) && isfinite(a.lo); }

__global__ void k_factor(const DevPlan P) {
    const int n_ent = P.tab_off[P.L + 2];
    const int idx = blockIdx.x * blockDim.x + threadIdx.x;
    if (idx >= n_ent) return;
    int l = 2;
    while (l < P.L + 1 && idx >= P.tab_off[l + 1]) ++l;
    const int r = idx - P.tab_off[l], n = P.nl[l];
    const int k = r / n, j = r - k * n;
    const double x = P.X[P.entry_off[l] + j];
    const dd wt = {P.Whi[P.entry_off[l] + j], P.Wlo[P.entry_off[l] + j]};
    const double ck = P.c[k];
    const dd xm = dd_from_sum(x, -0.5);   // x - 1/2 exactly
    dd Er = {1.0, 0.0}, Ei = {0.0, 0.0};
    switch (P.kind) {
    case SG_F_EXP_LINEAR:
        Er = dd_exp(dd_mul_d(xm, ck));
        break;
    case SG_F_OSCILLATORY: {
        // sincos of |a| with the sign applied afterwards: nodes placed symmetrically about 1/2 get
        // exactly conjugate factors (used by k_leaf2's symmetric-pair path)
        dd a = dd_mul_d(xm, ck), s, co;
        const bool neg = a.hi < 0.0;
        dd_sincos(neg ? dd_neg(a) : a, s, co);
        Er = co;
        Ei = neg ? dd_neg(s) : s;
        break;
    }
    case SG_F_GAUSSIAN: {
        // -c^2 ((x-w)^2 - (1/2-w)^2) = -c^2 (x - 1/2)(x + 1/2 - 2w)
        const double wk = P.w[k];
        dd xp = dd_add(dd_from_sum(x, 0.5), dd{-2.0 * wk, 0.0});
        dd arg = dd_mul(dd_mul(xm, xp), dd_from_prod(ck, ck));
        Er = dd_exp(dd_neg(arg));
        break;
    }
    case SG_F_PRODUCT_PEAK: {
        // phi(x)/phi(1/2) = (c^-2 + (1/2-w)^2) / (c^-2 + (x-w)^2)
        const double wk = P.w[k];
        dd ci2 = dd_div(dd{1.0, 0.0}, dd_from_prod(ck, ck));
        dd a = dd_from_sum(x, -wk), bm = dd_from_sum(0.5, -wk);
        Er = dd_div(dd_add(ci2, dd_mul(bm, bm)), dd_add(ci2, dd_mul(a, a)));
        break;
    }
    }
    dd Fr = dd_mul(wt, Er);
    P.Fre[idx] = make_double2(Fr.hi, Fr.lo);
    bool ok = dd_finite(Fr);
    if (P.kind == SG_F_OSCILLATORY) {
        dd Fi = dd_mul(wt, Ei);
        P.Fim[idx] = make_double2(Fi.hi, Fi.lo);
        ok = ok && dd_finite(Fi);
    }
    if (!ok) atomicOr(P.status, 1);
}

__global__ void __launch_bounds__(256) k_base(const DevPlan P) {
    // fixed-order strided partials, then a fixed CTA tree (sum; product for the peak kind)
    const bool prod = (P.kind == SG_F_PRODUCT_PEAK);
    dd acc = prod ? dd{1.0, 0.0} : dd{0.0, 0.0};
    for (int k = threadIdx.x; k < P.d; k += blockDim.x) {
        const double ck = P.c[k];
        switch (P.kind) {
        case SG_F_EXP_LINEAR:
        case SG_F_OSCILLATORY:
            acc = dd_add(acc, dd{0.5 * ck, 0.0});
            break;
        case SG_F_GAUSSIAN: {
            dd bm = dd_from_sum(0.5, -P.w[k]);
            acc = dd_add(acc, dd_mul(dd_mul(bm, bm), dd_from_prod(ck, ck)));
            break;
        }
        case SG_F_PRODUCT_PEAK: {
            dd bm = dd_from_sum(0.5, -P.w[k]);
            dd ci2 = dd_div(dd{1.0, 0.0}, dd_from_prod(ck, ck));
            acc = dd_mul(acc, dd_div(dd{1.0, 0.0}, dd_add(ci2, dd_mul(bm, bm))));
            break;
        }
        }
    }
    __shared__ double2 sm[256];
    sm[threadIdx.x] = make_double2(acc.hi, acc.lo);
    __syncthreads();
    for (int s = 128; s > 0; s >>= 1) {
        if (threadIdx.x < s) {
            dd a = {sm[threadIdx.x].x, sm[threadIdx.x].y}, b = {sm[threadIdx.x + s].x, sm[threadIdx.x + s].y};
            dd r = prod ? dd_mul(a, b) : dd_add(a, b);
            sm[threadIdx.x] = make_double2(r.hi, r.lo);
        }
        __syncthreads();
    }
    if (threadIdx.x == 0) {
        dd s = {sm[0].x, sm[0].y};
        dd Br = s, Bi = {0.0, 0.0};
        switch (P.kind) {
        case SG_F_EXP_LINEAR: Br = dd_exp(s); break;
        case SG_F_GAUSSIAN: Br = dd_exp(dd_neg(s)); break;
        case SG_F_PRODUCT_PEAK: Br = s; break;
        case SG_F_OSCILLATORY: {
            const double u = P.u[0];
            dd th = dd_add(dd_from_prod(DD_2PI_0, u), dd_from_prod(DD_2PI_1, u));
            th = dd_add(th, dd{DD_2PI_2 * u, 0.0});
            th = dd_add(th, s);
            dd sn, cs;
            dd_sincos(th, sn, cs);
            Br = cs;
            Bi = sn;
            break;
        }
        }
        P.base[0] = Br.hi;
        P.base[1] = Br.lo;
        P.base[2] = Bi.hi;
        P.base[3] = Bi.lo;
        if (!dd_finite(Br) || !dd_finite(Bi)) atomicOr(P.status, 1);
    }
}

// ---------------------------------------------------------------------------------------------
// leaf arithmetic helpers
// ---------------------------------------------------------------------------------------------
// acc (hi, lo) += p + e  : TwoSum on the high parts, plain sum of the low parts.
__device__ __forceinline__ void acc_add(double &ah, double &al, double p, double e) {
    double s = ah + p;
    double bb = s - ah;
    double err = (ah - (s - bb)) + (p - bb);
    al += err + e;
    ah = s;
}

// v * C(t, b): the node coefficient of depth t and excess b (an exact integer double unless merged)
__device__ __forceinline__ dd coef_mul(const DevPlan &P, dd v, int t, int b) {
    const double2 c = P.coefm[t * (P.L + 1) + b];
    return c.y == 0.0 ? dd_mul_d(v, c.x) : dd_mul(v, dd{c.x, c.y});
}

// ---------------------------------------------------------------------------------------------
// Root pass: every depth-1 point (k1, l1, j1) of this shard, one thread each.
// ---------------------------------------------------------------------------------------------
template <bool CPLX>
__global__ void __launch_bounds__(256) k_root(const DevPlan P, const RootArgs R) {
    const long long r1 = R.lo + (long long)blockIdx.x * blockDim.x + threadIdx.x;
    dd tot = {0.0, 0.0};
    if (r1 < R.hi) {
        const int k1 = (int)(r1 / P.M0);
        int rem = (int)(r1 - (long long)k1 * P.M0);
        int l1 = 2;
        while (rem >= P.nl[l1]) {
            rem -= P.nl[l1];
            ++l1;
        }
        const int j1 = rem;
        const int ti = P.tab_off[l1] + k1 * P.nl[l1] + j1;
        const dd Br = {P.base[0], P.base[1]};
        const double2 fr = P.Fre[ti];
        dd cr, ci = {0.0, 0.0};
        if (CPLX) {
            const dd Bi = {P.base[2], P.base[3]};
            const double2 fi = P.Fim[ti];
            cdd ch = cdd_mul(cdd{Br, Bi}, cdd{dd{fr.x, fr.y}, dd{fi.x, fi.y}});
            cr = ch.re;
            ci = ch.im;
        } else {
            cr = dd_mul(Br, dd{fr.x, fr.y});
        }
        const int b1 = l1 - 1;
        tot = coef_mul(P, cr, 1, b1);
        if (P.nfront >= 1 && b1 <= P.L - 1 && k1 <= P.d - 2) {
            const long long seg = (long long)b1 * P.d + k1;
            const long long o = R.off1[seg] + j1 - R.JS[seg];
            R.dst_re[o] = make_double2(cr.hi, cr.lo);
            if (CPLX) R.dst_im[o] = make_double2(ci.hi, ci.lo);
            R.dst_meta[o] = ((uint32_t)b1 << SG_META_KBITS) | (uint32_t)k1;
        }
    }
    dd s = block_reduce_dd<8>(tot);
    if (threadIdx.x == 0) R.partials[blockIdx.x] = make_double2(s.hi, s.lo);
}

// ---------------------------------------------------------------------------------------------
// Pass t >= 1 (K3 leaf + K2 frontier): warp task = (32 consecutive frontier-t nodes, a k' range).
// Lane = one parent prefix, held in registers; the loop over its children (k', l', j') reads the
// factor table at warp-uniform addresses (one broadcast transaction per load).
// ---------------------------------------------------------------------------------------------
#ifndef FOLD
#define FOLD 32   // rows between folds of acc_lo onto the grid (A/B: 32 vs 16: c5 -0.8%, c4 -1.4%; rel. error 2.7e-20 vs 1e-20)
#endif
#ifndef LEAF_MINB
#define LEAF_MINB 3
#endif

struct LeafAcc {
    double h, l;
};

// Biased grid accumulator (all leaf kernels).  The lane's high accumulator a.h starts at sigma =
// 1.5 * 2^m (2^m > 2 * bound on the sum of |P F| over the lane's children) and stays inside the
// binade [2^m, 2^(m+1)), where the double grid is u = ulp(sigma).  fma(P.hi, F.hi, a.h) therefore adds
// P.hi * F.hi rounded ONCE to the grid, exactly; the grid part h = new - old is exact (Sterbenz), and
// the remainder P.hi*F.hi - h (|.| <= u/2) and the cross terms P.hi*F.lo + P.lo*F.hi go to a.l by
// FMAs.  The lane result is (a.h - sigma) + a.l.  One FP64 instruction per product fewer than
// forming h = fma(P.hi, F.hi, sigma) - sigma and adding it.
template <bool CPLX>
__device__ __forceinline__ void leaf_term(const dd &er, const dd &ei, const double2 f, const double2 fi,
                                          LeafAcc &a) {
    if (!CPLX) {
        const double a1 = fma(er.hi, f.x, a.h);
        const double h = a1 - a.h;
        a.h = a1;
        a.l += fma(er.hi, f.x, -h);
        a.l = fma(er.hi, f.y, a.l);
        a.l = fma(er.lo, f.x, a.l);
    } else {
        // Re((er + i ei)(f + i fi)) = er f - ei fi, both grid parts added to a.h in turn
        const double a1 = fma(er.hi, f.x, a.h);
        const double h1 = a1 - a.h;
        const double a2 = fma(-ei.hi, fi.x, a1);
        const double h2 = a2 - a1;
        a.h = a2;
        a.l += fma(er.hi, f.x, -h1) + fma(-ei.hi, fi.x, -h2);
        a.l = fma(er.hi, f.y, a.l);
        a.l = fma(er.lo, f.x, a.l);
        a.l = fma(-ei.hi, fi.y, a.l);
        a.l = fma(-ei.lo, fi.x, a.l);
    }
}

__device__ __forceinline__ void leaf_fold(LeafAcc &a, double sigma) {
    const double t = (a.l + sigma) - sigma;
    a.h += t;
    a.l -= t;
}

#ifndef PASS_MINB
#define PASS_MINB 3   // CTAs/SM bound of k_pass
#endif
template <bool CPLX, bool WRITE>
__global__ void __launch_bounds__(PASS_THREADS, PASS_MINB) k_pass(const DevPlan P, const PassArgs A) {
    const int lane = threadIdx.x & 31, wib = threadIdx.x >> 5;
    const long long task = (long long)blockIdx.x * WPB + wib;
    dd tot = {0.0, 0.0};
    if (task < A.ntasks) {
        const int d = P.d, L = P.L;
        const long long chunk = task / A.nsplit;
        const int split = (int)(task - chunk * A.nsplit);
        const long long g = chunk * 32 + lane;
        const bool valid = g < A.nsrc;
        int b = L, k = d;
        dd pr = {0.0, 0.0}, pim = {0.0, 0.0};
        if (valid) {
            const uint32_t m = A.src_meta[g];
            b = (int)(m >> SG_META_KBITS);
            k = (int)(m & META_KMASK);
            const double2 v = A.src_re[g];
            pr = dd{v.x, v.y};
            if (CPLX) {
                const double2 vi = A.src_im[g];
                pim = dd{vi.x, vi.y};
            }
        }
        const int ks0 = (int)((long long)split * d / A.nsplit);
        const int ks1 = (int)((long long)(split + 1) * d / A.nsplit);
        const int kmin = __reduce_min_sync(0xffffffffu, valid ? k : INT_MAX);
        const int bmin = __reduce_min_sync(0xffffffffu, b);
        long long iseg = 0, Nseg = 0, Cseg = 0;
        if (WRITE && valid) {
            const long long s = (long long)b * d + k;
            iseg = g - A.offT[s];
            Nseg = A.NT[s];
            Cseg = A.CT[s];
        }
        const double pabs = fabs(pr.hi) + (CPLX ? fabs(pim.hi) : 0.0);
        const int kb = max(ks0, kmin + 1);
        for (int lp = 2; lp <= L + 1 - bmin; ++lp) {
            const bool lv = valid && (lp <= L + 1 - b);
            const int n = P.nl[lp];
            const int bp = b + lp - 1;
            const double2 *Fr = P.Fre + P.tab_off[lp];
            const double2 *Fi = CPLX ? P.Fim + P.tab_off[lp] : nullptr;
            const bool wr = WRITE && lv && (bp <= L - 1);
            const long long wbase = (long long)n * Cseg + iseg;
            // biased grid accumulator (leaf_term): sigma = 1.5 * 2^m > 2 * bound on the lane's
            // children of this level, from the suffix table SA
            const double bound = lv ? pabs * P.SA[(long long)lp * (d + 1) + min(k + 1, d)] * (1.0 + 0x1p-20) : 0.0;
            int ex = 0;
            frexp(2.0 * bound, &ex);
            const double sigma = bound > 0.0 ? ldexp(1.5, ex) : 1.5;
            LeafAcc acc = {sigma, 0.0};
            int nfold = 0;
            for (int kp = kb; kp < ks1; ++kp) {
                const bool kv = lv && (kp > k);
                const dd er = kv ? pr : dd{0.0, 0.0};
                const dd ei = kv ? pim : dd{0.0, 0.0};
                const bool wk = wr && kv && (kp <= d - 2);
                long long tb = 0;
                if (WRITE && wk) tb = A.TB[((long long)b * L + bp) * d + kp] + wbase;
                const double2 *fr_row = Fr + kp * n;
                const double2 *fi_row = CPLX ? Fi + kp * n : nullptr;
                for (int j = 0; j < n; ++j) {
                    const double2 f = __ldg(fr_row + j);
                    const double2 fi = CPLX ? __ldg(fi_row + j) : make_double2(0.0, 0.0);
                    leaf_term<CPLX>(er, ei, f, fi, acc);
                    if (WRITE && wk) {
                        // the stored child product P F in dd (complex for the oscillatory kind)
                        const long long o = tb + (long long)j * Nseg;
                        double p1, e1;
                        dd_mul_pe(er, dd{f.x, f.y}, p1, e1);
                        if (!CPLX) {
                            const dd ch = dd_norm(p1, e1);
                            A.dst_re[o] = make_double2(ch.hi, ch.lo);
                        } else {
                            double p2, e2, p3, e3, p4, e4;
                            dd_mul_pe(ei, dd{fi.x, fi.y}, p2, e2);
                            dd_mul_pe(er, dd{fi.x, fi.y}, p3, e3);
                            dd_mul_pe(ei, dd{f.x, f.y}, p4, e4);
                            const dd cre = dd_combine_pe(p1, e1, -p2, -e2), cim = dd_combine_pe(p3, e3, p4, e4);
                            A.dst_re[o] = make_double2(cre.hi, cre.lo);
                            A.dst_im[o] = make_double2(cim.hi, cim.lo);
                        }
                        A.dst_meta[o] = ((uint32_t)bp << SG_META_KBITS) | (uint32_t)kp;
                    }
                }
                if (++nfold == FOLD) {
                    nfold = 0;
                    leaf_fold(acc, sigma);
                }
            }
            if (lv) tot = dd_add(tot, coef_mul(P, dd_norm(acc.h - sigma, acc.l), A.t + 1, bp));
        }
    }
    dd s = block_reduce_dd<WPB>(tot);
    if (threadIdx.x == 0) A.partials[blockIdx.x] = make_double2(s.hi, s.lo);
}

// ---------------------------------------------------------------------------------------------
// Leaf-only pass (no extendable children): the hot loop of configs 4-5 (>= 97% of the points).
//
// Same task mapping as k_pass, but the accumulation is "grid-split": with sigma = 1.5 * 2^m and
// 2^m >= 2 * (bound on sum |P F| over the lane's children, from the suffix table SA), the high part
// h = fma(P.hi, F.hi, sigma) - sigma of every product is P.hi F.hi rounded once to the grid
// u = ulp(sigma), so acc_hi += h is EXACT; the remainder and the cross terms are small and go to
// acc_lo by FMAs (folded back onto the grid every FOLD rows).  7 FP64 instructions per real leaf
// and 14 per oscillatory leaf, against 12 / 24 with TwoSum + dd products.
// Children (k', j') are walked row by row (k'), NJ nodes per row unrolled with one accumulator pair
// per node for ILP; rows with k' <= max lane k of the warp are predicated (segment boundaries).
// ---------------------------------------------------------------------------------------------

// Leaf term for a node whose factor is REAL (imaginary part exactly 0): the midpoint node x = 1/2 of
// a level (E_k(1/2) = 1 for every kind, so F = w exactly real).  Re(P F) = P.re F: 7 FP64
// instructions instead of 14 for the oscillatory kind; bitwise the same value the general formula
// gives with F.im = 0 (every dropped term is an exact zero).
// CZ: the factor's low part is exactly 0 (combination form: F = w * 1), its cross term drops.
template <bool CZ = false>
__device__ __forceinline__ void leaf_real_factor_term(const dd &er, const double2 f, double &ah, double &al) {
    const double a1 = fma(er.hi, f.x, ah);   // biased accumulator (leaf_term)
    const double h = a1 - ah;
    ah = a1;
    double c = fma(er.lo, f.x, fma(er.hi, f.x, -h));
    if (!CZ) c = fma(er.hi, f.y, c);
    al += c;
}

// Symmetric pair (x_0 = 1 - x_2, w_0 = w_2; oscillatory): F_0 = conj(F_2) exactly, so the two
// points' terms Re(P F_0) = A + B and Re(P F_2) = A - B share the products A = P.re F_2.re and
// B = P.im F_2.im (their grid parts, remainders and cross terms); each point's term is still formed
// and accumulated on its own: node 0 adds the grid parts of A and B in turn (biased accumulator,
// leaf_term), node 2 forms h_A - h_B and adds it.  16 FP64 instructions for the two points.
__device__ __forceinline__ void leaf_sym_pair_terms(const dd &er, const dd &ei, const double2 f, const double2 g,
                                                    double &ah, double &al) {
    const double a1 = fma(er.hi, f.x, ah);
    const double h1 = a1 - ah;
    const double a2 = fma(ei.hi, g.x, a1);   // node 0: A + B
    const double h2 = a2 - a1;
    const double cA = fma(er.lo, f.x, fma(er.hi, f.y, fma(er.hi, f.x, -h1)));
    const double cB = fma(ei.lo, g.x, fma(ei.hi, g.y, fma(ei.hi, g.x, -h2)));
    al += cA + cB;
    ah = a2 + (h1 - h2);                     // node 2: A - B
    al += cA - cB;
}

template <bool CPLX, int NJ>
__device__ __forceinline__ void leaf_rows(const double2 *__restrict__ Fr, const double2 *__restrict__ Fi,
                                          int n, int kp0, int kp1, int klane, bool pred, const dd &pr,
                                          const dd &pim, double sigma, LeafAcc (&acc)[NJ > 0 ? NJ : 1]) {
    const int nj = NJ > 0 ? NJ : n;
    for (int kp = kp0; kp < kp1;) {
        const int ke = min(kp1, kp + FOLD);
        for (; kp < ke; ++kp) {
            const bool kv = !pred || kp > klane;
            const dd er = kv ? pr : dd{0.0, 0.0};
            const dd ei = (CPLX && kv) ? pim : dd{0.0, 0.0};
            const double2 *fr = Fr + (long long)kp * nj;
            const double2 *fi = CPLX ? Fi + (long long)kp * nj : nullptr;
            if (NJ > 0) {
#pragma unroll
                for (int j = 0; j < (NJ > 0 ? NJ : 1); ++j) {
                    const double2 f = __ldg(fr + j);
                    const double2 g = CPLX ? __ldg(fi + j) : make_double2(0.0, 0.0);
                    leaf_term<CPLX>(er, ei, f, g, acc[j]);
                }
            } else {
                for (int j = 0; j < nj; ++j) {
                    const double2 f = __ldg(fr + j);
                    const double2 g = CPLX ? __ldg(fi + j) : make_double2(0.0, 0.0);
                    leaf_term<CPLX>(er, ei, f, g, acc[0]);
                }
            }
        }
#pragma unroll
        for (int j = 0; j < (NJ > 0 ? NJ : 1); ++j) leaf_fold(acc[j], sigma);
    }
}

template <bool CPLX, int NJ>
__device__ __forceinline__ dd leaf_level(const double2 *Fr, const double2 *Fi, int n, int kb, int kmain,
                                         int ks1, int k, const dd &pr, const dd &pim, double sigma) {
    LeafAcc acc[NJ > 0 ? NJ : 1];
#pragma unroll
    for (int j = 0; j < (NJ > 0 ? NJ : 1); ++j) acc[j] = LeafAcc{sigma, 0.0};   // biased accumulator
    // boundary rows (some lanes of the warp have k >= k'), then the unpredicated main rows
    leaf_rows<CPLX, NJ>(Fr, Fi, n, kb, min(kmain, ks1), k, true, pr, pim, sigma, acc);
    leaf_rows<CPLX, NJ>(Fr, Fi, n, max(kb, kmain), ks1, k, false, pr, pim, sigma, acc);
    dd s = {0.0, 0.0};
#pragma unroll
    for (int j = 0; j < (NJ > 0 ? NJ : 1); ++j) s = dd_add(s, dd_norm(acc[j].h - sigma, acc[j].l));
    return s;
}

// Symmetric oscillatory row of NJ nodes: pairs (j, NJ-1-j) share their products
// (leaf_sym_pair_terms, F_j = conj(F_{NJ-1-j})), the midpoint's factor (odd NJ) is real; one biased
// accumulator pair per pair plus one for the midpoint.  8 FP64 instructions per point for even NJ
// (midpoint-merged rows), 7.0 for NJ = 3, 7.4 for NJ = 5, instead of 12.
#ifndef LEAF_SYM_SPLIT
#define LEAF_SYM_SPLIT 0   // 1: the two nodes of a pair in separate accumulators (shorter chains)
#endif
#define LEAF_SYM_NACC(NJ) (LEAF_SYM_SPLIT ? NJ : (NJ + 1) / 2)
// node 0 (A + B) into accumulator a, node 2 (A - B) into b
__device__ __forceinline__ void leaf_sym_pair_split(const dd &er, const dd &ei, const double2 f, const double2 g,
                                                    LeafAcc &a, LeafAcc &b) {
    const double u1 = fma(er.hi, f.x, a.h);
    const double h1 = u1 - a.h;
    a.h = fma(ei.hi, g.x, u1);
    const double h2 = a.h - u1;
    const double cA = fma(er.lo, f.x, fma(er.hi, f.y, fma(er.hi, f.x, -h1)));
    const double cB = fma(ei.lo, g.x, fma(ei.hi, g.y, fma(ei.hi, g.x, -h2)));
    a.l += cA + cB;
    b.h += h1 - h2;
    b.l += cA - cB;
}

template <int NJ>
__device__ __forceinline__ void leaf_rows_sym(const double2 *__restrict__ Fr, const double2 *__restrict__ Fi,
                                              int kp0, int kp1, int klane, bool pred, const dd &pr, const dd &pim,
                                              double sigma, LeafAcc (&acc)[LEAF_SYM_NACC(NJ)]) {
    constexpr int NP = NJ / 2;
    for (int kp = kp0; kp < kp1;) {
        const int ke = min(kp1, kp + FOLD);
        for (; kp < ke; ++kp) {
            const bool kv = !pred || kp > klane;
            const dd er = kv ? pr : dd{0.0, 0.0};
            const dd ei = kv ? pim : dd{0.0, 0.0};
            const double2 *fr = Fr + (long long)kp * NJ;
            const double2 *fi = Fi + (long long)kp * NJ;
#pragma unroll
            for (int q = 0; q < NP; ++q) {
                if constexpr (LEAF_SYM_SPLIT)
                    leaf_sym_pair_split(er, ei, __ldg(fr + NJ - 1 - q), __ldg(fi + NJ - 1 - q), acc[q], acc[NJ - 1 - q]);
                else
                    leaf_sym_pair_terms(er, ei, __ldg(fr + NJ - 1 - q), __ldg(fi + NJ - 1 - q), acc[q].h, acc[q].l);
            }
            if constexpr (NJ % 2 == 1) leaf_real_factor_term<false>(er, __ldg(fr + NP), acc[NP].h, acc[NP].l);
        }
#pragma unroll
        for (int q = 0; q < LEAF_SYM_NACC(NJ); ++q) leaf_fold(acc[q], sigma);
    }
}

template <int NJ>
__device__ __forceinline__ dd leaf_level_sym(const double2 *Fr, const double2 *Fi, int kb, int kmain, int ks1,
                                             int k, const dd &pr, const dd &pim, double sigma) {
    LeafAcc acc[LEAF_SYM_NACC(NJ)];
#pragma unroll
    for (int q = 0; q < LEAF_SYM_NACC(NJ); ++q) acc[q] = LeafAcc{sigma, 0.0};   // biased accumulator
    leaf_rows_sym<NJ>(Fr, Fi, kb, min(kmain, ks1), k, true, pr, pim, sigma, acc);
    leaf_rows_sym<NJ>(Fr, Fi, max(kb, kmain), ks1, k, false, pr, pim, sigma, acc);
    dd s = {0.0, 0.0};
#pragma unroll
    for (int q = 0; q < LEAF_SYM_NACC(NJ); ++q) s = dd_add(s, dd_norm(acc[q].h - sigma, acc[q].l));
    return s;
}

template <bool CPLX>
__global__ void __launch_bounds__(PASS_THREADS, LEAF_MINB) k_leaf(const DevPlan P, const PassArgs A) {
    const int lane = threadIdx.x & 31, wib = threadIdx.x >> 5;
    const long long task = (long long)blockIdx.x * WPB + wib;
    dd tot = {0.0, 0.0};
    if (task < A.ntasks) {
        const int d = P.d, L = P.L;
        const long long chunk = task / A.nsplit;
        const int split = (int)(task - chunk * A.nsplit);
        const long long g = chunk * 32 + lane;
        const bool valid = g < A.nsrc;
        int b = L, k = d;
        dd pr = {0.0, 0.0}, pim = {0.0, 0.0};
        if (valid) {
            const uint32_t m = A.src_meta[g];
            b = (int)(m >> SG_META_KBITS);
            k = (int)(m & META_KMASK);
            const double2 v = A.src_re[g];
            pr = dd{v.x, v.y};
            if (CPLX) {
                const double2 vi = A.src_im[g];
                pim = dd{vi.x, vi.y};
            }
        }
        const int ks0 = (int)((long long)split * d / A.nsplit);
        const int ks1 = (int)((long long)(split + 1) * d / A.nsplit);
        const int kmin = __reduce_min_sync(0xffffffffu, valid ? k : INT_MAX);
        const int kmax = __reduce_max_sync(0xffffffffu, valid ? k : -1);
        const int bmin = __reduce_min_sync(0xffffffffu, b);
        const int kb = max(ks0, kmin + 1), kmain = kmax + 1;
        const double pabs = fabs(pr.hi) + (CPLX ? fabs(pim.hi) : 0.0);
        for (int lp = 2; lp <= L + 1 - bmin; ++lp) {
            const bool lv = valid && (lp <= L + 1 - b);
            const dd er = lv ? pr : dd{0.0, 0.0};
            const dd ei = lv ? pim : dd{0.0, 0.0};
            const int n = P.nl[lp];
            // sigma = 1.5 * 2^m with 2^m >= 2 * bound on sum |p| over this lane's children
            const double bound = lv ? pabs * P.SA[(long long)lp * (d + 1) + min(k + 1, d)] * (1.0 + 0x1p-20) : 0.0;
            int ex = 0;
            frexp(2.0 * bound, &ex);
            const double sigma = bound > 0.0 ? ldexp(1.5, ex) : 1.5;
            const double2 *Fr = P.Fre + P.tab_off[lp];
            const double2 *Fi = CPLX ? P.Fim + P.tab_off[lp] : nullptr;
            dd s;
            const bool sym = CPLX && ((P.symmask >> lp) & 1);
            if (sym && n == 3) s = leaf_level_sym<3>(Fr, Fi, kb, kmain, ks1, k, er, ei, sigma);
            else if (sym && n == 5) s = leaf_level_sym<5>(Fr, Fi, kb, kmain, ks1, k, er, ei, sigma);
            else if (sym && n == 2) s = leaf_level_sym<2>(Fr, Fi, kb, kmain, ks1, k, er, ei, sigma);
            else if (sym && n == 4) s = leaf_level_sym<4>(Fr, Fi, kb, kmain, ks1, k, er, ei, sigma);
            else switch (n) {
            case 2: s = leaf_level<CPLX, 2>(Fr, Fi, n, kb, kmain, ks1, k, er, ei, sigma); break;
            case 3: s = leaf_level<CPLX, 3>(Fr, Fi, n, kb, kmain, ks1, k, er, ei, sigma); break;
#ifdef LEAF_NJ5
            case 5: s = leaf_level<CPLX, 5>(Fr, Fi, n, kb, kmain, ks1, k, er, ei, sigma); break;
#endif
            default: s = leaf_level<CPLX, 0>(Fr, Fi, n, kb, kmain, ks1, k, er, ei, sigma); break;
            }
            if (lv) tot = dd_add(tot, coef_mul(P, s, A.t + 1, b + lp - 1));
        }
    }
    dd s = block_reduce_dd<WPB>(tot);
    if (threadIdx.x == 0) A.partials[blockIdx.x] = make_double2(s.hi, s.lo);
}

// ---------------------------------------------------------------------------------------------
// k_leaf1: the last pass when every source prefix has excess L-1 (t = L-1), so every child has
// level 2 and coefficient coef[L]: the dominant kernel of configs 4-5 (c4: 99.6%, c5: 97.4% of the
// points).  Lean register budget (<= 64 -> 32 warps/SM), one accumulator pair per lane with short
// dependency chains, two rows (k', k'+1) per iteration for ILP.  Oscillatory leaf = 14 FP64
// instructions: h1, h2 (4), acc.h += h1 + h2 (2), remainder t1 + cross-term FMA chain (5),
// remainder t2 (1), acc.l (2); real leaf = 7.
// ---------------------------------------------------------------------------------------------
template <bool CPLX>
__device__ __forceinline__ void leaf1_term(const dd &er, const dd &ei, const double2 f, const double2 fi,
                                           double &ah, double &al) {
    // biased accumulator ah (see leaf_term); the remainder t = P.hi F.hi - h (one rounding) seeds the
    // FMA chain of the cross terms.  Real: 6 FP64 instructions (4 DFMA + 2 DADD); oscillatory: 12.
    if (!CPLX) {
        const double a1 = fma(er.hi, f.x, ah);
        const double h = a1 - ah;
        ah = a1;
        double c = fma(er.lo, f.x, fma(er.hi, f.x, -h));
        c = fma(er.hi, f.y, c);
        al += c;
    } else {
        const double a1 = fma(er.hi, f.x, ah);
        const double h1 = a1 - ah;
        const double a2 = fma(-ei.hi, fi.x, a1);
        const double h2 = a2 - a1;
        ah = a2;
        double c = fma(er.lo, f.x, fma(er.hi, f.x, -h1));
        c = fma(er.hi, f.y, c);
        c = fma(-ei.lo, fi.x, c);
        c = fma(-ei.hi, fi.y, c);
        al += c + fma(-ei.hi, fi.x, -h2);
    }
}

#ifndef LEAF1_MINB
#define LEAF1_MINB 4
#endif
#ifndef LEAF1_PERJ
#define LEAF1_PERJ 0   // 1 = one accumulator pair per node j of the row (measured slower)
#endif
#ifndef LEAF1_ROWS
#define LEAF1_ROWS 4   // rows k' per loop iteration (A/B: 4 > 2 > 1)
#endif

template <bool CPLX, int NJ, int NA, bool SMEM>
__device__ __forceinline__ void leaf1_row(const double2 *__restrict__ Fr, const double2 *__restrict__ Fi, int kp,
                                          const dd &er, const dd &ei, double (&ah)[NA], double (&al)[NA]) {
    double2 f[NJ], g[NJ];
#pragma unroll
    for (int j = 0; j < NJ; ++j) {
        f[j] = SMEM ? Fr[kp * NJ + j] : __ldg(Fr + kp * NJ + j);
        g[j] = CPLX ? (SMEM ? Fi[kp * NJ + j] : __ldg(Fi + kp * NJ + j)) : make_double2(0.0, 0.0);
    }
#pragma unroll
    for (int j = 0; j < NJ; ++j) leaf1_term<CPLX>(er, ei, f[j], g[j], ah[j % NA], al[j % NA]);
}

// One warp task of the single-level leaf pass: returns this lane's coefficient-free sum.
template <bool CPLX, int NJ, bool SMEM>
__device__ __forceinline__ dd leaf1_task(const DevPlan &P, const PassArgs &A, long long task,
                                         const double2 *Fr, const double2 *Fi) {
    constexpr int NA = LEAF1_PERJ ? NJ : 1;
    const int lane = threadIdx.x & 31;
    const int d = P.d;
    const long long chunk = task / A.nsplit;
    const int split = (int)(task - chunk * A.nsplit);
    const long long g = chunk * 32 + lane;
    const bool valid = g < A.nsrc;
    int k = d;
    dd pr = {0.0, 0.0}, pim = {0.0, 0.0};
    if (valid) {
        k = (int)(A.src_meta[g] & META_KMASK);
        const double2 v = A.src_re[g];
        pr = dd{v.x, v.y};
        if (CPLX) {
            const double2 vi = A.src_im[g];
            pim = dd{vi.x, vi.y};
        }
    }
    const int ks0 = (int)((long long)split * d / A.nsplit);
    const int ks1 = (int)((long long)(split + 1) * d / A.nsplit);
    const int kmin = __reduce_min_sync(0xffffffffu, valid ? k : INT_MAX);
    const int kmax = __reduce_max_sync(0xffffffffu, valid ? k : -1);
    const int kb = max(ks0, kmin + 1);
    const double bound = valid ? (fabs(pr.hi) + (CPLX ? fabs(pim.hi) : 0.0)) *
                                     P.SA[2LL * (d + 1) + min(k + 1, d)] * (1.0 + 0x1p-20)
                               : 0.0;
    int ex = 0;
    frexp(2.0 * bound, &ex);
    const double sigma = bound > 0.0 ? ldexp(1.5, ex) : 1.5;
    double ah[NA], al[NA];
#pragma unroll
    for (int a = 0; a < NA; ++a) {
        ah[a] = sigma;   // biased accumulator
        al[a] = 0.0;
    }
    // boundary rows: lanes whose prefix ends at k >= k' contribute zero
    const int kmid = min(kmax + 1, ks1);
    for (int kp = kb; kp < kmid; ++kp) {
        const bool kv = kp > k;
        const dd er = kv ? pr : dd{0.0, 0.0};
        const dd ei = kv ? pim : dd{0.0, 0.0};
        leaf1_row<CPLX, NJ, NA, SMEM>(Fr, Fi, kp, er, ei, ah, al);
    }
    // main rows, LEAF1_ROWS per iteration, folded back onto the grid every FOLD rows
    int kp = max(kb, kmid);
    while (kp < ks1) {
        const int ke = min(ks1, kp + FOLD);
        for (; kp + LEAF1_ROWS - 1 < ke; kp += LEAF1_ROWS) {
#pragma unroll
            for (int r = 0; r < LEAF1_ROWS; ++r)
                leaf1_row<CPLX, NJ, NA, SMEM>(Fr, Fi, kp + r, pr, pim, ah, al);
        }
        for (; kp < ke; ++kp) leaf1_row<CPLX, NJ, NA, SMEM>(Fr, Fi, kp, pr, pim, ah, al);
#pragma unroll
        for (int a = 0; a < NA; ++a) {
            const double t = (al[a] + sigma) - sigma;
            ah[a] += t;
            al[a] -= t;
        }
    }
    dd s = {0.0, 0.0};
    if (valid) {
#pragma unroll
        for (int a = 0; a < NA; ++a) s = dd_add(s, dd_from_sum(ah[a] - sigma, al[a]));
    }
    return s;
}

// Persistent: gridDim.x = resident CTAs; CTA c's warp w runs tasks (c*WPB + w) + i*gridDim.x*WPB
// (static round robin over tasks sorted heavy-first, so partials stay deterministic).  With SMEM the
// level-2 factor slice (d x NJ entries) is staged once per CTA in shared memory, so the warp-uniform
// row loads are broadcast LDS instead of LDG through the L1 data path.
template <bool CPLX, int NJ, bool SMEM>
__global__ void __launch_bounds__(PASS_THREADS, LEAF1_MINB) k_leaf1(const DevPlan P, const PassArgs A) {
    extern __shared__ double2 fsm[];
    const int wib = threadIdx.x >> 5;
    const double2 *Fr = P.Fre + P.tab_off[2];
    const double2 *Fi = CPLX ? P.Fim + P.tab_off[2] : nullptr;
    if (SMEM) {
        const int n = P.d * NJ;
        for (int i = threadIdx.x; i < n; i += blockDim.x) {
            fsm[i] = Fr[i];
            if (CPLX) fsm[n + i] = Fi[i];
        }
        __syncthreads();
        Fr = fsm;
        Fi = CPLX ? fsm + n : nullptr;
    }
    (void)wib;
    const int lane = threadIdx.x & 31;
    // dynamic scheduling: warps pull tasks (sorted heavy-first) from a global counter; every task
    // writes its own partial, so the fixed-order reduction keeps results bitwise reproducible
    for (;;) {
        unsigned long long task = 0;
        if (lane == 0) task = atomicAdd(A.counter, 1ull);
        task = __shfl_sync(0xffffffffu, task, 0);
        if ((long long)task >= A.ntasks) break;
        dd v = warp_reduce_dd(leaf1_task<CPLX, NJ, SMEM>(P, A, (long long)task, Fr, Fi));
        if (lane == 0) {
            v = dd_mul_d(v, P.coef[P.L]);
            A.partials[task] = make_double2(v.hi, v.lo);
        }
    }
}

// ---------------------------------------------------------------------------------------------
// k_leaf2: fused last two levels.  The depth-(L-1) prefixes are never stored: a warp task is
// (k_mid, 32 stored depth-(L-2) parents of excess L-2 whose last active coordinate is < k_mid);
// each lane forms P' = P * F[2][k_mid][j_mid] in full double-double for every node j_mid, then
// walks the rows k' > k_mid of its level-2 children exactly like k_leaf1.  All lanes share k_mid,
// so every row is warp-uniform (no boundary predication).  Saves the write + read of frontier
// L-1 (config 5: 119 M nodes, 4.3 GB each way).
// ---------------------------------------------------------------------------------------------
struct Leaf2Args {
    const double2 *src_re, *src_im;   // frontier L-2
    long long base;                   // offset of segment (b = L-2, k = 0) in frontier L-2
    const long long *Cmid;            // C_{L-2}(L-2, k): parents of excess L-2 with k_last < k
    const long long *T2;              // task descriptors: first parent, (ka << 32) | kb (plan.h)
    long long ntasks;
    double2 *partials;             // one per task
    unsigned long long *counter;   // dynamic task counter, zeroed per launch
};

#ifndef LEAF2_ROWS
#define LEAF2_ROWS 1        // rows per iteration, real kinds (A/B on config 4: 1 > 2)
#endif
#ifndef LEAF2_ROWS_CPLX
#define LEAF2_ROWS_CPLX 4   // rows per iteration, oscillatory (A/B on config 5: 4 = 6 = 8 > 2 > 1)
#endif
#ifndef LEAF2_MINB
#define LEAF2_MINB 3        // CTAs/SM bound, real kinds (80 regs)
#endif
#ifndef LEAF2_MINB_CPLX
#define LEAF2_MINB_CPLX 2   // CTAs/SM bound, oscillatory (108 regs, 16 warps/SM: 26.14 ms vs 27.52)
#endif

// CJ = index of the midpoint node in the level-2 row (-1: none), fixed per launch by the host;
// SYM: nodes 0 and 2 form a symmetric pair (CJ == 1, NJ == 3, oscillatory), or nodes 0 and 1 do
// (CJ == -1, NJ == 2: the midpoint-merged Clenshaw-Curtis level-2 row {0, 1}).
#ifndef LEAF2_SPLITR
#define LEAF2_SPLITR 0  // same split for the real kinds' NJ = 3 row with midpoint
#endif
#ifndef LEAF2_SPLIT2
#define LEAF2_SPLIT2 1  // same split for the midpoint-merged NJ = 2 symmetric row (merged c5 -0.6%)
#endif
#ifndef LEAF2_SPLIT
#define LEAF2_SPLIT 1   // second accumulator pair per mid (node 2 + midpoint): shorter chains, c5 -1%
#endif
template <bool CPLX, int NJ, bool SMEM, int CJ, bool SYM = false, bool CZ = false>
__device__ __forceinline__ void leaf2_row_multi(const double2 *__restrict__ Fr, const double2 *__restrict__ Fi,
                                                int kp, const dd (&er)[NJ], const dd (&ei)[NJ],
                                                double (&ah)[NJ], double (&al)[NJ], double (&bh)[NJ],
                                                double (&bl)[NJ]) {
    if constexpr (LEAF2_SPLIT && SYM && CPLX && NJ == 3 && CJ == 1) {
        const double2 f2 = SMEM ? Fr[kp * 3 + 2] : __ldg(Fr + kp * 3 + 2);
        const double2 g2 = SMEM ? Fi[kp * 3 + 2] : __ldg(Fi + kp * 3 + 2);
        const double2 f1 = SMEM ? Fr[kp * 3 + 1] : __ldg(Fr + kp * 3 + 1);
#pragma unroll
        for (int jm = 0; jm < 3; ++jm) {
            // node 0 (A + B) into accumulator a, node 2 (A - B) and the midpoint into b
            const double u1 = fma(er[jm].hi, f2.x, ah[jm]);
            const double h1 = u1 - ah[jm];
            ah[jm] = fma(ei[jm].hi, g2.x, u1);
            const double h2 = ah[jm] - u1;
            const double cA = fma(er[jm].lo, f2.x, fma(er[jm].hi, f2.y, fma(er[jm].hi, f2.x, -h1)));
            const double cB = fma(ei[jm].lo, g2.x, fma(ei[jm].hi, g2.y, fma(ei[jm].hi, g2.x, -h2)));
            al[jm] += cA + cB;
            bh[jm] += h1 - h2;
            bl[jm] += cA - cB;
            leaf_real_factor_term<CZ>(er[jm], f1, bh[jm], bl[jm]);
        }
        return;
    }
    if constexpr (SYM && CPLX && NJ == 3 && CJ == 1) {
        const double2 f2 = SMEM ? Fr[kp * 3 + 2] : __ldg(Fr + kp * 3 + 2);
        const double2 g2 = SMEM ? Fi[kp * 3 + 2] : __ldg(Fi + kp * 3 + 2);
        const double2 f1 = SMEM ? Fr[kp * 3 + 1] : __ldg(Fr + kp * 3 + 1);
#pragma unroll
        for (int jm = 0; jm < 3; ++jm) {
            leaf_sym_pair_terms(er[jm], ei[jm], f2, g2, ah[jm], al[jm]);
            leaf_real_factor_term<CZ>(er[jm], f1, ah[jm], al[jm]);
        }
        return;
    }
    if constexpr (SYM && CPLX && NJ == 2 && CJ == -1) {
        const double2 f1 = SMEM ? Fr[kp * 2 + 1] : __ldg(Fr + kp * 2 + 1);
        const double2 g1 = SMEM ? Fi[kp * 2 + 1] : __ldg(Fi + kp * 2 + 1);
#pragma unroll
        for (int jm = 0; jm < 2; ++jm) {
            if constexpr (LEAF2_SPLIT2) {
                // node 0 (A + B) into accumulator a, node 1 (A - B) into b: shorter chains
                const double u1 = fma(er[jm].hi, f1.x, ah[jm]);
                const double h1 = u1 - ah[jm];
                ah[jm] = fma(ei[jm].hi, g1.x, u1);
                const double h2 = ah[jm] - u1;
                const double cA = fma(er[jm].lo, f1.x, fma(er[jm].hi, f1.y, fma(er[jm].hi, f1.x, -h1)));
                const double cB = fma(ei[jm].lo, g1.x, fma(ei[jm].hi, g1.y, fma(ei[jm].hi, g1.x, -h2)));
                al[jm] += cA + cB;
                bh[jm] += h1 - h2;
                bl[jm] += cA - cB;
            } else {
                leaf_sym_pair_terms(er[jm], ei[jm], f1, g1, ah[jm], al[jm]);
            }
        }
        return;
    }
    double2 f[NJ], g[NJ];
#pragma unroll
    for (int j = 0; j < NJ; ++j) {
        f[j] = SMEM ? Fr[kp * NJ + j] : __ldg(Fr + kp * NJ + j);
        g[j] = (CPLX && j != CJ) ? (SMEM ? Fi[kp * NJ + j] : __ldg(Fi + kp * NJ + j)) : make_double2(0.0, 0.0);
    }
#pragma unroll
    for (int j = 0; j < NJ; ++j)
#pragma unroll
        for (int jm = 0; jm < NJ; ++jm) {
            if constexpr (LEAF2_SPLITR && !CPLX && NJ == 3 && CJ == 1) {
                // real kinds: node 0 and the midpoint into accumulator a, node 2 into b
                if (j == CJ) leaf_real_factor_term<CZ>(er[jm], f[j], ah[jm], al[jm]);
                else if (j == 0) leaf1_term<CPLX>(er[jm], ei[jm], f[j], g[j], ah[jm], al[jm]);
                else leaf1_term<CPLX>(er[jm], ei[jm], f[j], g[j], bh[jm], bl[jm]);
                continue;
            }
            if (j == CJ) leaf_real_factor_term<CZ>(er[jm], f[j], ah[jm], al[jm]);
            else leaf1_term<CPLX>(er[jm], ei[jm], f[j], g[j], ah[jm], al[jm]);
        }
}

template <bool CPLX, int NJ, bool SMEM, int CJ, bool SYM = false, bool CZ = false>
__global__ void __launch_bounds__(PASS_THREADS, CPLX ? LEAF2_MINB_CPLX : LEAF2_MINB) k_leaf2(const DevPlan P, const Leaf2Args A) {
    extern __shared__ double2 fsm[];
    const int lane = threadIdx.x & 31, wib = threadIdx.x >> 5;
    const int d = P.d;
    const double2 *Fr = P.Fre + P.tab_off[2];
    const double2 *Fi = CPLX ? P.Fim + P.tab_off[2] : nullptr;
    if (SMEM) {
        const int n = d * NJ;
        for (int i = threadIdx.x; i < n; i += blockDim.x) {
            fsm[i] = Fr[i];
            if (CPLX) fsm[n + i] = Fi[i];
        }
        __syncthreads();
        Fr = fsm;
        Fi = CPLX ? fsm + n : nullptr;
    }
    (void)wib;
    for (;;) {
        unsigned long long utask = 0;
        if (lane == 0) utask = atomicAdd(A.counter, 1ull);
        utask = __shfl_sync(0xffffffffu, utask, 0);
        const long long task = (long long)utask;
        if (task >= A.ntasks) break;
        // task = (chunk of 32 parents starting at `first`, k_mid range [ka, kb)), plan.h T2
        const long long first = A.T2[2 * task], kk = A.T2[2 * task + 1];
        const int ka = (int)(kk >> 32), kb = (int)(kk & 0xffffffffLL);
        const long long i = first + lane;
        dd pr = {0.0, 0.0}, pim = {0.0, 0.0};
        if (i < A.Cmid[kb - 1]) {   // Cmid is nondecreasing: valid for the last k_mid
            const double2 v = A.src_re[A.base + i];
            pr = dd{v.x, v.y};
            if (CPLX) {
                const double2 vi = A.src_im[A.base + i];
                pim = dd{vi.x, vi.y};
            }
        }
        dd lane_sum = {0.0, 0.0};
        for (int km = ka; km < kb; ++km) {
            const bool valid = i < A.Cmid[km];
            const dd prv = valid ? pr : dd{0.0, 0.0};
            const dd pimv = valid ? pim : dd{0.0, 0.0};
            const double sa = P.SA[2LL * (d + 1) + km + 1] * (1.0 + 0x1p-20);
            // all NJ mid prefixes of the lane at once: NJ independent accumulator chains that share
            // every row load (ILP x NJ, shared-memory loads / leaf / NJ)
            dd er[NJ], ei[NJ];
            double sg[NJ], ah[NJ], al[NJ], bh[NJ], bl[NJ];
            if constexpr (CPLX && SYM && NJ == 3 && CJ == 1) {
                // mids 0 and 2 are conjugate (F_0 = conj(F_2)): P F_2 and P conj(F_2) share their
                // four products; mid 1 (the midpoint) is real
                const double2 f = Fr[km * 3 + 2], g = Fi[km * 3 + 2], w1 = Fr[km * 3 + 1];
                cdd c2, c0;
                cdd_mul_conj_pair(cdd{prv, pimv}, cdd{dd{f.x, f.y}, dd{g.x, g.y}}, c2, c0);
                er[0] = c0.re;
                ei[0] = c0.im;
                er[2] = c2.re;
                ei[2] = c2.im;
                er[1] = CZ ? dd_mul_d(prv, w1.x) : dd_mul(prv, dd{w1.x, w1.y});
                ei[1] = CZ ? dd_mul_d(pimv, w1.x) : dd_mul(pimv, dd{w1.x, w1.y});
            } else if constexpr (CPLX && SYM && NJ == 2 && CJ == -1) {
                const double2 f = Fr[km * 2 + 1], g = Fi[km * 2 + 1];
                cdd c1, c0;
                cdd_mul_conj_pair(cdd{prv, pimv}, cdd{dd{f.x, f.y}, dd{g.x, g.y}}, c1, c0);
                er[0] = c0.re;
                ei[0] = c0.im;
                er[1] = c1.re;
                ei[1] = c1.im;
            } else {
#pragma unroll
                for (int jm = 0; jm < NJ; ++jm) {
                    const double2 f = Fr[km * NJ + jm];
                    if (CPLX) {
                        const double2 g = Fi[km * NJ + jm];
                        cdd c = cdd_mul_fast(cdd{prv, pimv}, cdd{dd{f.x, f.y}, dd{g.x, g.y}});
                        er[jm] = c.re;
                        ei[jm] = c.im;
                    } else {
                        er[jm] = dd_mul(prv, dd{f.x, f.y});
                        ei[jm] = dd{0.0, 0.0};
                    }
                }
            }
#pragma unroll
            for (int jm = 0; jm < NJ; ++jm) {
                const double bound = (fabs(er[jm].hi) + (CPLX ? fabs(ei[jm].hi) : 0.0)) * sa;
                int ex = 0;
                frexp(2.0 * bound, &ex);
                sg[jm] = bound > 0.0 ? ldexp(1.5, ex) : 1.5;
                ah[jm] = sg[jm];   // biased accumulator
                al[jm] = 0.0;
                bh[jm] = sg[jm];
                bl[jm] = 0.0;
            }
            int kp = km + 1;
            while (kp < d) {
                const int ke = min(d, kp + FOLD);
                constexpr int RW = CPLX ? LEAF2_ROWS_CPLX : LEAF2_ROWS;
                for (; kp + RW - 1 < ke; kp += RW) {
#pragma unroll
                    for (int r = 0; r < RW; ++r)
                        leaf2_row_multi<CPLX, NJ, SMEM, CJ, SYM, CZ>(Fr, Fi, kp + r, er, ei, ah, al, bh, bl);
                }
                for (; kp < ke; ++kp) leaf2_row_multi<CPLX, NJ, SMEM, CJ, SYM, CZ>(Fr, Fi, kp, er, ei, ah, al, bh, bl);
#pragma unroll
                for (int jm = 0; jm < NJ; ++jm) {
                    if ((LEAF2_SPLIT && SYM && CPLX && NJ == 3 && CJ == 1) ||
                        (LEAF2_SPLIT2 && SYM && CPLX && NJ == 2 && CJ == -1) ||
                        (LEAF2_SPLITR && !CPLX && NJ == 3 && CJ == 1))
                        al[jm] += bl[jm], bl[jm] = 0.0;
                    const double t = (al[jm] + sg[jm]) - sg[jm];
                    ah[jm] += t;
                    al[jm] -= t;
                }
            }
            // lane value = sum_jm (ah - sigma) + al: exact grid parts via TwoSum, low parts in FP64
            if ((LEAF2_SPLIT && SYM && CPLX && NJ == 3 && CJ == 1) ||
                (LEAF2_SPLIT2 && SYM && CPLX && NJ == 2 && CJ == -1) ||
                (LEAF2_SPLITR && !CPLX && NJ == 3 && CJ == 1)) {
#pragma unroll
                for (int jm = 0; jm < NJ; ++jm) {   // same grid, |sum| < 2^m: exact
                    ah[jm] += bh[jm] - sg[jm];
                    al[jm] += bl[jm];
                }
            }
            double hs = ah[0] - sg[0], ls = al[0];
#pragma unroll
            for (int jm = 1; jm < NJ; ++jm) {
                double e;
                two_sum(hs, ah[jm] - sg[jm], hs, e);
                ls += al[jm] + e;
            }
            lane_sum = dd_add_fast(lane_sum, dd_norm(hs, ls));
        }
        dd v = warp_reduce_dd_fast(lane_sum);
        if (lane == 0) {
            v = dd_mul_d(v, P.coef[P.L]);
            A.partials[task] = make_double2(v.hi, v.lo);
        }
    }
}

// ---------------------------------------------------------------------------------------------
// s-form: the literal "partial sums carried one coordinate at a time, outer function applied at the
// leaf" design (§8f row 4).  A node carries delta = sum_active a_k(x_k) and its
// weight product W; a leaf evaluates g(S + delta') once per point and accumulates c(e) W' g in dd.
//   SG_ARITH_SFORM_FP64 (DDS = false): delta and g in FP64 (CUDA exp/cos/pow) — the ablation that
//     measures what per-point FP64 outer functions cost and lose (not parity-grade).
//   SG_ARITH_SFORM_DD (DDS = true): delta, S and g in double-double (dd exp / sincos / powers) —
//     parity-grade, and the only path for integrands that are NOT products of per-coordinate
//     factors: the Genz corner peak g(s) = (1 + s)^-(d+1) of s = sum c_k x_k.
// Kinds: exp / Gaussian g = exp(S + delta) (Gaussian a_k = -c_k^2 ((x-w_k)^2 - (1/2-w_k)^2)),
// oscillatory g = cos(S + delta) (S includes 2 pi u), corner peak g = (S + delta)^-(d+1) with
// S = 1 + sum c_k / 2.  Tables reuse the factor-table slots: Fre[idx] = weight (dd),
// Fim[idx] = a (dd; lo = 0 in FP64 mode); base[0..1] = S (dd); frontier re = W, im = delta.
// ---------------------------------------------------------------------------------------------
template <bool DDS>
__global__ void k_factor_s(const DevPlan P) {
    const int n_ent = P.tab_off[P.L + 2];
    const int idx = blockIdx.x * blockDim.x + threadIdx.x;
    if (idx >= n_ent) return;
    int l = 2;
    while (l < P.L + 1 && idx >= P.tab_off[l + 1]) ++l;
    const int r = idx - P.tab_off[l], n = P.nl[l];
    const int k = r / n, j = r - k * n;
    const double x = P.X[P.entry_off[l] + j];
    const double ck = P.c[k];
    dd a;
    if (P.kind == SG_F_GAUSSIAN) {
        const double wk = P.w[k];
        if (DDS) {
            // -c^2 ((x-w)^2 - (1/2-w)^2) = -c^2 (x - 1/2)(x + 1/2 - 2w)
            const dd xm = dd_from_sum(x, -0.5);
            const dd xp = dd_add(dd_from_sum(x, 0.5), dd{-2.0 * wk, 0.0});
            a = dd_neg(dd_mul(dd_mul(xm, xp), dd_from_prod(ck, ck)));
        } else {
            a = dd{-(ck * ck) * ((x - wk) * (x - wk) - (0.5 - wk) * (0.5 - wk)), 0.0};
        }
    } else {
        a = DDS ? dd_mul_d(dd_from_sum(x, -0.5), ck) : dd{ck * (x - 0.5), 0.0};
    }
    P.Fre[idx] = make_double2(P.Whi[P.entry_off[l] + j], P.Wlo[P.entry_off[l] + j]);
    P.Fim[idx] = make_double2(a.hi, a.lo);
    if (!isfinite(a.hi)) atomicOr(P.status, 1);
}

// S in dd: fixed-order strided partials, then a fixed CTA tree (deterministic)
__global__ void __launch_bounds__(256) k_base_s(const DevPlan P) {
    dd acc = {0.0, 0.0};
    double cneg = 0.0;   // corner peak: sum of negative c_k (domain 1 + sum min(c_k, 0) > 0)
    for (int k = threadIdx.x; k < P.d; k += blockDim.x) {
        const double ck = P.c[k];
        cneg += ck < 0.0 ? ck : 0.0;
        if (P.kind == SG_F_GAUSSIAN) {
            const dd bm = dd_from_sum(0.5, -P.w[k]);
            acc = dd_sub(acc, dd_mul(dd_mul(bm, bm), dd_from_prod(ck, ck)));
        } else {
            acc = dd_add(acc, dd{0.5 * ck, 0.0});
        }
    }
    __shared__ double2 sm[256];
    __shared__ double sneg[256];
    sm[threadIdx.x] = make_double2(acc.hi, acc.lo);
    sneg[threadIdx.x] = cneg;
    __syncthreads();
    for (int st = 128; st > 0; st >>= 1) {
        if (threadIdx.x < st) {
            const dd r = dd_add(dd{sm[threadIdx.x].x, sm[threadIdx.x].y}, dd{sm[threadIdx.x + st].x, sm[threadIdx.x + st].y});
            sm[threadIdx.x] = make_double2(r.hi, r.lo);
            sneg[threadIdx.x] += sneg[threadIdx.x + st];
        }
        __syncthreads();
    }
    if (threadIdx.x == 0 && P.kind == SG_F_CORNER_PEAK && !(1.0 + sneg[0] > 0.0)) atomicOr(P.status, 1);
    if (threadIdx.x == 0) {
        dd S = {sm[0].x, sm[0].y};
        if (P.kind == SG_F_OSCILLATORY) {
            const double u = P.u[0];
            dd th = dd_add(dd_from_prod(DD_2PI_0, u), dd_from_prod(DD_2PI_1, u));
            th = dd_add(th, dd{DD_2PI_2 * u, 0.0});
            S = dd_add(S, th);
        }
        if (P.kind == SG_F_CORNER_PEAK) S = dd_add(S, dd{1.0, 0.0});
        P.base[0] = S.hi;
        P.base[1] = S.lo;
        P.base[2] = 0.0;
        P.base[3] = 0.0;
        if (!dd_finite(S)) atomicOr(P.status, 1);
    }
}

__device__ __forceinline__ double sform_g(int kind, int d, double arg) {
    if (kind == SG_F_OSCILLATORY) return cos(arg);
    if (kind == SG_F_CORNER_PEAK) return pow(arg, -(double)(d + 1));
    return exp(arg);
}

// y^n, n >= 1, by binary powering in dd (left-to-right; ~2 log2 n products)
__device__ __forceinline__ dd dd_powi(dd y, int n) {
    int top = 31 - __clz(n);
    dd r = y;
    for (int bit = top - 1; bit >= 0; --bit) {
        r = dd_mul(r, r);
        if ((n >> bit) & 1) r = dd_mul(r, y);
    }
    return r;
}

__device__ __forceinline__ dd sform_g_dd(int kind, int d, dd y) {
    if (kind == SG_F_OSCILLATORY) {
        dd sn, cs;
        dd_sincos(y, sn, cs);
        return cs;
    }
    if (kind == SG_F_CORNER_PEAK) return dd_powi(dd_recip(y), d + 1);
    return dd_exp(y);
}

template <bool DDS>
__device__ __forceinline__ dd sform_value(const DevPlan &P, dd arg) {
    return DDS ? sform_g_dd(P.kind, P.d, arg) : dd{sform_g(P.kind, P.d, arg.hi), 0.0};
}

template <bool DDS>
__global__ void __launch_bounds__(256) k_root_s(const DevPlan P, const RootArgs R) {
    const long long r1 = R.lo + (long long)blockIdx.x * blockDim.x + threadIdx.x;
    dd tot = {0.0, 0.0};
    if (r1 < R.hi) {
        const int k1 = (int)(r1 / P.M0);
        int rem = (int)(r1 - (long long)k1 * P.M0);
        int l1 = 2;
        while (rem >= P.nl[l1]) {
            rem -= P.nl[l1];
            ++l1;
        }
        const int j1 = rem;
        const int ti = P.tab_off[l1] + k1 * P.nl[l1] + j1;
        const double2 wv = P.Fre[ti], av = P.Fim[ti];
        const dd W = {wv.x, wv.y}, delta = {av.x, av.y};
        const dd S = {P.base[0], P.base[1]};
        const dd arg = DDS ? dd_add(S, delta) : dd{S.hi + delta.hi, 0.0};
        const int b1 = l1 - 1;
        tot = dd_mul_d(dd_mul(W, sform_value<DDS>(P, arg)), P.coef[b1]);
        if (P.nfront >= 1 && b1 <= P.L - 1 && k1 <= P.d - 2) {
            const long long seg = (long long)b1 * P.d + k1;
            const long long o = R.off1[seg] + j1 - R.JS[seg];
            R.dst_re[o] = wv;
            R.dst_im[o] = av;
            R.dst_meta[o] = ((uint32_t)b1 << SG_META_KBITS) | (uint32_t)k1;
        }
    }
    dd s = block_reduce_dd<8>(tot);
    if (threadIdx.x == 0) R.partials[blockIdx.x] = make_double2(s.hi, s.lo);
}

template <bool DDS, bool WRITE>
__global__ void __launch_bounds__(PASS_THREADS) k_pass_s(const DevPlan P, const PassArgs A) {
    const int lane = threadIdx.x & 31, wib = threadIdx.x >> 5;
    const long long task = (long long)blockIdx.x * WPB + wib;
    dd tot = {0.0, 0.0};
    if (task < A.ntasks) {
        const int d = P.d, L = P.L;
        const long long chunk = task / A.nsplit;
        const int split = (int)(task - chunk * A.nsplit);
        const long long g = chunk * 32 + lane;
        const bool valid = g < A.nsrc;
        int b = L, k = d;
        dd W = {0.0, 0.0}, delta = {0.0, 0.0};
        if (valid) {
            const uint32_t m = A.src_meta[g];
            b = (int)(m >> SG_META_KBITS);
            k = (int)(m & META_KMASK);
            const double2 v = A.src_re[g], dv = A.src_im[g];
            W = dd{v.x, v.y};
            delta = dd{dv.x, dv.y};
        }
        const int ks0 = (int)((long long)split * d / A.nsplit);
        const int ks1 = (int)((long long)(split + 1) * d / A.nsplit);
        const int kmin = __reduce_min_sync(0xffffffffu, valid ? k : INT_MAX);
        const int bmin = __reduce_min_sync(0xffffffffu, b);
        long long iseg = 0, Nseg = 0, Cseg = 0;
        if (WRITE && valid) {
            const long long s = (long long)b * d + k;
            iseg = g - A.offT[s];
            Nseg = A.NT[s];
            Cseg = A.CT[s];
        }
        const dd S = {P.base[0], P.base[1]};
        const int kb = max(ks0, kmin + 1);
        for (int lp = 2; lp <= L + 1 - bmin; ++lp) {
            const bool lv = valid && (lp <= L + 1 - b);
            const int n = P.nl[lp];
            const int bp = b + lp - 1;
            const double2 *Wt = P.Fre + P.tab_off[lp];
            const double2 *At = P.Fim + P.tab_off[lp];
            const bool wr = WRITE && lv && (bp <= L - 1);
            const long long wbase = (long long)n * Cseg + iseg;
            double ah = 0.0, al = 0.0;
            for (int kp = kb; kp < ks1; ++kp) {
                const bool kv = lv && (kp > k);
                const bool wk = wr && kv && (kp <= d - 2);
                long long tb = 0;
                if (WRITE && wk) tb = A.TB[((long long)b * L + bp) * d + kp] + wbase;
                for (int j = 0; j < n; ++j) {
                    const double2 wv = __ldg(Wt + kp * n + j), av = __ldg(At + kp * n + j);
                    // partial sum carried one coordinate further: dd (DDS) or FP64 (ablation)
                    const dd dl = DDS ? dd_add(delta, dd{av.x, av.y}) : dd{delta.hi + av.x, 0.0};
                    const dd Wc = dd_mul(W, dd{wv.x, wv.y});
                    dd gv = {0.0, 0.0};
                    if (kv) gv = sform_value<DDS>(P, DDS ? dd_add(S, dl) : dd{S.hi + dl.hi, 0.0});
                    double p, e;
                    dd_mul_pe(Wc, gv, p, e);
                    acc_add(ah, al, p, e);
                    if (WRITE && wk) {
                        const long long o = tb + (long long)j * Nseg;
                        A.dst_re[o] = make_double2(Wc.hi, Wc.lo);
                        A.dst_im[o] = make_double2(dl.hi, dl.lo);
                        A.dst_meta[o] = ((uint32_t)bp << SG_META_KBITS) | (uint32_t)kp;
                    }
                }
            }
            if (lv) tot = dd_add(tot, dd_mul_d(dd_norm(ah, al), P.coef[bp]));
        }
    }
    dd s = block_reduce_dd<WPB>(tot);
    if (threadIdx.x == 0) A.partials[blockIdx.x] = make_double2(s.hi, s.lo);
}

// SA[l][k] = sum_{k' >= k} sum_j (|Fre[l][k'][j].hi| + |Fim[l][k'][j].hi|): bound used by k_leaf.
// One CTA per level: chunked row sums, a serial suffix scan over the 256 chunk sums, then each
// thread writes the suffix values of its chunk (all loads in parallel; deterministic order).
__global__ void __launch_bounds__(256) k_suffix_abs(const DevPlan P) {
    const int l = 2 + blockIdx.x;
    if (l > P.L + 1) return;
    const int d = P.d, n = P.nl[l];
    const double2 *Fr = P.Fre + P.tab_off[l];
    const double2 *Fi = P.kind == SG_F_OSCILLATORY ? P.Fim + P.tab_off[l] : nullptr;
    const int chunk = (d + blockDim.x - 1) / blockDim.x;
    const int k0 = min(d, (int)threadIdx.x * chunk), k1 = min(d, k0 + chunk);
    auto row = [&](int k) {
        double r = 0.0;
        for (int j = 0; j < n; ++j) {
            r += fabs(Fr[(long long)k * n + j].x);
            if (Fi) r += fabs(Fi[(long long)k * n + j].x);
        }
        return r;
    };
    double cs = 0.0;
    for (int k = k0; k < k1; ++k) cs += row(k);
    __shared__ double suf[257];
    suf[threadIdx.x] = cs;
    __syncthreads();
    if (threadIdx.x == 0) {
        double run = 0.0;
        suf[blockDim.x] = 0.0;
        for (int i = blockDim.x - 1; i >= 0; --i) {
            const double v = suf[i];
            suf[i] = run;   // sum of the chunks after chunk i
            run += v;
        }
    }
    __syncthreads();
    double s = suf[threadIdx.x];
    if (threadIdx.x == 0) P.SA[(long long)l * (d + 1) + d] = 0.0;
    for (int k = k1 - 1; k >= k0; --k) {
        s += row(k);
        P.SA[(long long)l * (d + 1) + k] = s;
    }
}

// Level-1 reduction: block b sums partials [b*RED_CHUNK, (b+1)*RED_CHUNK) in a fixed order.
#define RED_CHUNK 8192
__global__ void __launch_bounds__(256) k_reduce_l1(const double2 *partials, long long n, double2 *out) {
    const long long b0 = (long long)blockIdx.x * RED_CHUNK, b1 = min(n, b0 + RED_CHUNK);
    dd s = {0.0, 0.0};
    for (long long i = b0 + threadIdx.x; i < b1; i += blockDim.x) s = dd_add(s, dd{partials[i].x, partials[i].y});
    s = block_reduce_dd<8>(s);
    if (threadIdx.x == 0) out[blockIdx.x] = make_double2(s.hi, s.lo);
}

// Final fixed-order reduction of the level-1 partials (+ the root point) -> out[0..1].
__global__ void __launch_bounds__(1024) k_reduce(const DevPlan P, const double2 *partials,
                                                 long long n, int include_root, double *out) {
    dd s = {0.0, 0.0};
    for (long long i = threadIdx.x; i < n; i += blockDim.x) s = dd_add(s, dd{partials[i].x, partials[i].y});
    s = block_reduce_dd<32>(s);
    if (threadIdx.x == 0) {
        if (include_root && P.coefm[0].x != 0.0) {
            const dd root = P.sform == 2   ? sform_g_dd(P.kind, P.d, dd{P.base[0], P.base[1]})
                            : P.sform == 1 ? dd{sform_g(P.kind, P.d, P.base[0]), 0.0}
                                           : dd{P.base[0], P.base[1]};
            s = dd_add(s, coef_mul(P, root, 0, 0));
        }
        if (*P.status) s = dd{nan(""), nan("")};
        out[0] = s.hi;
        out[1] = s.lo;
    }
}

// ---------------------------------------------------------------------------------------------
// Separable collapse (SG_METHOD_COLLAPSE): the paper's symbolic partial
// function f_{t-m} in its strongest form.  Because every integrand in scope
// is Re(B * prod_k E_k(x_k)), the sum over all tensor points of all multi-indices of one excess e
// factorises per coordinate:
//     sum_{|i| = d+e} (U^{i_1} x ... x U^{i_d}) (prod_k E_k) = [z^e] prod_k p_k(z),
//     p_k(z) = sum_{l=1}^{L+1} T_k(l) z^{l-1},  T_k(l) = sum_j F[l][k][j] = sum_j w_j^l E_k(x_j^l)
// (T_k(1) = 1: the midpoint, weight 1, E_k(1/2) = 1), so
//     A(q,d) f = Re(B * sum_e coef[e] [z^e] prod_k p_k(z))      (Eq 2.6; delta form: coef = 1 and
// the delta-form table F already holds Delta^l weights).  O(d L^2) dd work instead of O(points).
// Pass 1: CTA g multiplies the polynomials of a contiguous coordinate chunk (each thread its own
// contiguous sub-chunk, then a fixed pairwise tree in shared memory) -> one partial polynomial.
// Pass 2 (one CTA): fixed tree over the partials, coefficient dot product, times B, real part.
// Every product is taken in a fixed order: bitwise reproducible.
// ---------------------------------------------------------------------------------------------
#define COLLAPSE_THREADS 128
#define COLLAPSE_MAXB 148

// acc(z) <- acc(z) * p(z) mod z^{L+1}, in place (descending e: acc[e - i], i >= 1, is still old)
template <bool CPLX>
__device__ __forceinline__ void poly_mul_inplace(double2 *acc_re, double2 *acc_im, const double2 *p_re,
                                                 const double2 *p_im, int L) {
    for (int e = L; e >= 0; --e) {
        dd sr = {0.0, 0.0}, si = {0.0, 0.0};
        for (int i = 0; i <= e; ++i) {
            const dd ar = {acc_re[e - i].x, acc_re[e - i].y}, pr = {p_re[i].x, p_re[i].y};
            if (CPLX) {
                const dd ai = {acc_im[e - i].x, acc_im[e - i].y}, pi = {p_im[i].x, p_im[i].y};
                const cdd m = cdd_mul(cdd{ar, ai}, cdd{pr, pi});
                sr = dd_add(sr, m.re);
                si = dd_add(si, m.im);
            } else {
                sr = dd_add(sr, dd_mul(ar, pr));
            }
        }
        acc_re[e] = make_double2(sr.hi, sr.lo);
        if (CPLX) acc_im[e] = make_double2(si.hi, si.lo);
    }
}

// Shared-memory layout of pass 1/2: poly[thread][e] (re), then (im) — (L+1) double2 per thread each.
template <bool CPLX>
__device__ void collapse_tree(double2 *sre, double2 *sim, int L) {
    const int n1 = L + 1;
    for (int s = COLLAPSE_THREADS / 2; s > 0; s >>= 1) {
        __syncthreads();
        if ((int)threadIdx.x < s) {
            const int a = threadIdx.x, b = threadIdx.x + s;
            poly_mul_inplace<CPLX>(sre + a * n1, CPLX ? sim + a * n1 : nullptr, sre + b * n1,
                                   CPLX ? sim + b * n1 : nullptr, L);
        }
    }
    __syncthreads();
}

template <bool CPLX>
__global__ void __launch_bounds__(COLLAPSE_THREADS) k_collapse_part(const DevPlan P, double2 *part_re,
                                                                     double2 *part_im) {
    extern __shared__ double2 csm[];
    const int L = P.L, n1 = L + 1, d = P.d;
    double2 *sre = csm, *sim = csm + COLLAPSE_THREADS * n1;
    double2 *pre = csm + (CPLX ? 2 : 1) * COLLAPSE_THREADS * n1;   // this thread's p_k scratch
    double2 *pim = pre + COLLAPSE_THREADS * n1;
    double2 *are = sre + threadIdx.x * n1, *aim = sim + threadIdx.x * n1;
    double2 *qre = pre + threadIdx.x * n1, *qim = pim + threadIdx.x * n1;
    for (int e = 0; e < n1; ++e) {
        are[e] = make_double2(e == 0 ? 1.0 : 0.0, 0.0);
        if (CPLX) aim[e] = make_double2(0.0, 0.0);
    }
    // coordinate chunk of this CTA, sub-chunk of this thread (both contiguous, fixed)
    const long long g0 = (long long)d * blockIdx.x / gridDim.x, g1 = (long long)d * (blockIdx.x + 1) / gridDim.x;
    const long long n = g1 - g0;
    const int k0 = (int)(g0 + n * threadIdx.x / COLLAPSE_THREADS);
    const int k1 = (int)(g0 + n * (threadIdx.x + 1) / COLLAPSE_THREADS);
    for (int k = k0; k < k1; ++k) {
        qre[0] = make_double2(1.0, 0.0);
        if (CPLX) qim[0] = make_double2(0.0, 0.0);
        for (int l = 2; l <= L + 1; ++l) {
            const int nl = P.nl[l];
            const double2 *Fr = P.Fre + P.tab_off[l] + (long long)k * nl;
            const double2 *Fi = CPLX ? P.Fim + P.tab_off[l] + (long long)k * nl : nullptr;
            dd tr = {0.0, 0.0}, ti = {0.0, 0.0};
            for (int j = 0; j < nl; ++j) {
                tr = dd_add(tr, dd{Fr[j].x, Fr[j].y});
                if (CPLX) ti = dd_add(ti, dd{Fi[j].x, Fi[j].y});
            }
            qre[l - 1] = make_double2(tr.hi, tr.lo);
            if (CPLX) qim[l - 1] = make_double2(ti.hi, ti.lo);
        }
        poly_mul_inplace<CPLX>(are, aim, qre, qim, L);
    }
    collapse_tree<CPLX>(sre, sim, L);
    if (threadIdx.x == 0) {
        for (int e = 0; e < n1; ++e) {
            part_re[blockIdx.x * n1 + e] = sre[e];
            if (CPLX) part_im[blockIdx.x * n1 + e] = sim[e];
        }
    }
}

template <bool CPLX>
__global__ void __launch_bounds__(COLLAPSE_THREADS) k_collapse_final(const DevPlan P, const double2 *part_re,
                                                                      const double2 *part_im, int nparts,
                                                                      int emit, double *out) {
    extern __shared__ double2 csm[];
    const int L = P.L, n1 = L + 1;
    double2 *sre = csm, *sim = csm + COLLAPSE_THREADS * n1;
    for (int e = 0; e < n1; ++e) {
        const bool have = (int)threadIdx.x < nparts;
        sre[threadIdx.x * n1 + e] = have ? part_re[threadIdx.x * n1 + e] : make_double2(e == 0 ? 1.0 : 0.0, 0.0);
        if (CPLX) sim[threadIdx.x * n1 + e] = have ? part_im[threadIdx.x * n1 + e] : make_double2(0.0, 0.0);
    }
    // partials beyond the first COLLAPSE_THREADS fold into thread (i mod COLLAPSE_THREADS), in order
    for (int i = threadIdx.x + COLLAPSE_THREADS; i < nparts; i += COLLAPSE_THREADS)
        poly_mul_inplace<CPLX>(sre + threadIdx.x * n1, CPLX ? sim + threadIdx.x * n1 : nullptr, part_re + i * n1,
                               CPLX ? part_im + i * n1 : nullptr, L);
    collapse_tree<CPLX>(sre, sim, L);
    if (threadIdx.x == 0) {
        dd sr = {0.0, 0.0}, si = {0.0, 0.0};
        for (int e = 0; e <= L; ++e) {
            if (P.coef[e] == 0.0) continue;
            sr = dd_add(sr, dd_mul_d(dd{sre[e].x, sre[e].y}, P.coef[e]));
            if (CPLX) si = dd_add(si, dd_mul_d(dd{sim[e].x, sim[e].y}, P.coef[e]));
        }
        const dd Br = {P.base[0], P.base[1]}, Bi = {P.base[2], P.base[3]};
        dd a = CPLX ? dd_sub(dd_mul(Br, sr), dd_mul(Bi, si)) : dd_mul(Br, sr);
        if (!emit) a = dd{0.0, 0.0};   // ranks != 0 contribute nothing (the collapse is not sharded)
        if (*P.status || !dd_finite(a)) {
            atomicOr(P.status, 1);
            a = dd{nan(""), nan("")};
        }
        out[0] = a.hi;
        out[1] = a.lo;
    }
}

__global__ void k_finalize(const double *gathered, int world, const int *status, double *result) {
    if (threadIdx.x != 0 || blockIdx.x != 0) return;
    dd s = {0.0, 0.0};
    for (int r = 0; r < world; ++r) s = dd_add(s, dd{gathered[2 * r], gathered[2 * r + 1]});
    if (*status || !isfinite(s.hi)) s = dd{nan(""), nan("")};
    result[0] = s.hi;
    result[1] = s.lo;
}

// ---------------------------------------------------------------------------------------------
// plan object and C ABI
// ---------------------------------------------------------------------------------------------
struct sg_plan_s {
    HostPlan hp;
    DevPlan dp;
    bool cplx = false;
    bool sform = false;        // s-form kernels (SG_ARITH_SFORM_FP64 or SG_ARITH_SFORM_DD)
    bool sform_dd = false;     // SG_ARITH_SFORM_DD: dd partial sums and outer function
    bool two = false;          // frontier layout with a second double2 array (complex or s-form)
    bool collapse = false;     // SG_METHOD_COLLAPSE: O(d L^2) per-coordinate polynomial product
    int collapse_blocks = 0;   // CTAs of k_collapse_part (one partial polynomial each)
    bool collapse_emit = true; // rank 0 emits the value; other ranks contribute 0
    // plan-owned device memory
    void *dev_block = nullptr;
    size_t dev_bytes = 0;
    long long *d_tabs = nullptr;
    std::vector<size_t> tab_offT, tab_NT, tab_CT, tab_TB;   // element offsets into d_tabs per depth
    size_t tab_JS = 0, tab_off1 = 0, tab_TK = 0;
    double *d_scratch = nullptr;   // 4 doubles
    // profiling hook (sg_profile_enable): events around every launch of sg_integrate
    bool prof = false;
    // specialised single-level leaf kernel (k_leaf1); SG_B200_GENERIC_LEAF=1 forces k_leaf (tests)
    bool leaf1 = true;
    int leaf1_t = -1;          // pass index run by the persistent k_leaf1 / k_leaf2 (or -1)
    bool leaf2 = false;        // last two levels fused (hp.fuse): k_leaf2
    long long leaf1_grid = 0;  // persistent grid (resident CTAs) of k_leaf1 / k_leaf2
    bool leaf2_center = false; // level-2 row has its midpoint at index 1 (real oscillatory factor)
    bool leaf2_sym = false;    // level-2 nodes 0 and 2 symmetric about 1/2 (conjugate factors)
    bool leaf2_cz = false;     // midpoint factor has an exactly zero low part (combination form)
    unsigned long long *d_counter = nullptr;   // dynamic task counter (plan-owned)
    size_t leaf1_smem = 0;     // its dynamic shared memory (0 = factor rows read through L1)
    std::vector<cudaEvent_t> ev;
    // workspace
    char *ws = nullptr;
    size_t ws_bytes = 0;
    size_t ws_front_off[2] = {0, 0}, ws_part_off = 0, ws_red_off = 0, ws_need = 0;
};

static size_t align_up(size_t x, size_t a) { return (x + a - 1) / a * a; }
static int setup_leaf1(sg_plan_s *p);

static bool finite_array(const double *a, int n) {
    for (int i = 0; i < n; ++i)
        if (!isfinite(a[i])) return false;
    return true;
}

static int validate_desc(const sg_integrand_desc *f, int d) {
    if (!f || !f->c) return SG_EINVAL;
    if (f->d != d) return SG_EINVAL;
    if ((int)f->kind < 0 || (int)f->kind > 4) return SG_EINVAL;
    if ((f->kind == SG_F_PRODUCT_PEAK || f->kind == SG_F_GAUSSIAN) && !f->w) return SG_EINVAL;
    return SG_OK;
}

// corner peak: 1 + sum c_k x_k > 0 on the whole cube (its minimum is 1 + sum min(c_k, 0))
static bool corner_domain_ok(const double *c, int d) {
    double m = 1.0;
    for (int k = 0; k < d; ++k) m += c[k] < 0.0 ? c[k] : 0.0;
    return m > 0.0;
}

extern "C" const char *sg_strerror(int code) {
    switch (code) {
    case SG_OK: return "ok";
    case SG_EINVAL: return "invalid argument (bad pointer/enum/size, q < d, non-finite parameter)";
    case SG_EUNSUPPORTED: return "unsupported level or size";
    case SG_EOVERFLOW: return "point or frontier count overflows 63 bits";
    case SG_ENOMEM: return "out of device memory or workspace too small";
    case SG_ECUDA: return "CUDA runtime error";
    case SG_ENONFINITE: return "non-finite integrand value";
    case SG_ENOWORKSPACE: return "no workspace attached";
    }
    return "unknown status";
}

extern "C" int sg_plan(int d, int q, sg_rule rule, const sg_integrand_desc *f, const sg_options *opt,
                       sg_plan_t *out) {
    if (!out) return SG_EINVAL;
    *out = nullptr;
    if (d < 1 || q < d) return SG_EINVAL;
    int rc = validate_desc(f, d);
    if (rc) return rc;
    if (!finite_array(f->c, d)) return SG_EINVAL;
    if (f->w && (f->kind == SG_F_PRODUCT_PEAK || f->kind == SG_F_GAUSSIAN) && !finite_array(f->w, d))
        return SG_EINVAL;
    if (!isfinite(f->u)) return SG_EINVAL;
    if (f->kind == SG_F_PRODUCT_PEAK)
        for (int k = 0; k < d; ++k)
            if (f->c[k] == 0.0) return SG_EINVAL;
    if (f->kind == SG_F_CORNER_PEAK && !corner_domain_ok(f->c, d)) return SG_EINVAL;
    sg_options o = {SG_FORM_COMBINATION, SG_ARITH_FACTOR_DD, 0, 1, 0, -1};
    if (opt) o = *opt;
    if (o.arith != SG_ARITH_FACTOR_DD && o.arith != SG_ARITH_SFORM_FP64 && o.arith != SG_ARITH_SFORM_DD)
        return SG_EINVAL;
    // the corner peak is not a product of per-coordinate factors: no factor table exists, its
    // parity-grade path is the dd s-form (collapse and merge need the factor form)
    if (f->kind == SG_F_CORNER_PEAK && o.method == SG_METHOD_COLLAPSE) return SG_EUNSUPPORTED;
    if (f->kind == SG_F_CORNER_PEAK && o.arith == SG_ARITH_FACTOR_DD) o.arith = SG_ARITH_SFORM_DD;
    if (o.arith != SG_ARITH_FACTOR_DD && f->kind == SG_F_PRODUCT_PEAK) return SG_EUNSUPPORTED;
    if (o.merge != SG_MERGE_NONE && o.merge != SG_MERGE_MIDPOINT) return SG_EINVAL;
    if (o.merge != SG_MERGE_NONE && o.arith != SG_ARITH_FACTOR_DD) return SG_EUNSUPPORTED;
    if (o.method != SG_METHOD_TREE && o.method != SG_METHOD_COLLAPSE) return SG_EINVAL;
    if (o.method == SG_METHOD_COLLAPSE) {
        if (o.merge != SG_MERGE_NONE) return SG_EINVAL;
        if (o.arith != SG_ARITH_FACTOR_DD) return SG_EUNSUPPORTED;
        if (o.world < 1 || o.rank < 0 || o.rank >= o.world) return SG_EINVAL;
    }
    sg_plan_s *p = new (std::nothrow) sg_plan_s();
    if (!p) return SG_ENOMEM;
    {
        // SG_B200_NOFUSE=1 / SG_B200_FUSE=1 override the automatic choice (tests, A/B runs)
        const char *nf = getenv("SG_B200_NOFUSE"), *fu = getenv("SG_B200_FUSE");
        int mode = (nf && nf[0] == '1') ? 0 : (fu && fu[0] == '1') ? 2 : 1;
        if (o.arith != SG_ARITH_FACTOR_DD) mode = 0;
        if (o.method == SG_METHOD_COLLAPSE) {
            // whole problem on every rank (the collapse is not sharded); no tree passes run
            p->collapse = true;
            p->collapse_emit = (o.rank == 0);
            rc = host_plan_build(p->hp, d, q - d, (int)rule, (int)f->kind, (int)o.form, 0, 0, 1, 0, -1, 0);
        } else {
            rc = host_plan_build(p->hp, d, q - d, (int)rule, (int)f->kind, (int)o.form, (int)o.merge, o.rank,
                                 o.world, o.range_lo, o.range_hi, mode);
        }
    }
    if (rc) {
        delete p;
        return rc;
    }
    HostPlan &hp = p->hp;
    p->cplx = (f->kind == SG_F_OSCILLATORY);
    p->sform = (o.arith == SG_ARITH_SFORM_FP64 || o.arith == SG_ARITH_SFORM_DD);
    p->sform_dd = (o.arith == SG_ARITH_SFORM_DD);
    p->two = p->cplx || p->sform;
    if (p->sform) p->leaf1 = false;
    {
        const char *g = getenv("SG_B200_GENERIC_LEAF");
        p->leaf1 = !(g && g[0] == '1');
    }
    // ---- device tables: one allocation ----
    const int L = hp.L, nent = (int)hp.X.size();
    std::vector<long long> tabs;
    p->tab_offT.assign(hp.nfront + 2, 0);
    p->tab_NT.assign(hp.nfront + 2, 0);
    p->tab_CT.assign(hp.nfront + 2, 0);
    p->tab_TB.assign(hp.nfront + 2, 0);
    auto push = [&](const std::vector<int64_t> &v) {
        size_t o = tabs.size();
        tabs.insert(tabs.end(), v.begin(), v.end());
        return o;
    };
    for (int t = 1; t <= hp.nfront; ++t) {
        p->tab_offT[t] = push(hp.off[t]);
        p->tab_NT[t] = push(hp.N[t]);
        p->tab_CT[t] = push(hp.C[t]);
        if (t < hp.nfront) p->tab_TB[t] = push(hp.TB[t]);
    }
    p->tab_JS = push(hp.JS);
    if (hp.fuse) p->tab_TK = push(hp.T2);
    p->tab_off1 = hp.nfront >= 1 ? p->tab_offT[1] : 0;
    if (tabs.empty()) tabs.push_back(0);
    size_t sz = 0;
    auto carve = [&](size_t bytes) {
        size_t o = sz;
        sz = align_up(sz + bytes, 256);
        return o;
    };
    const size_t oX = carve(sizeof(double) * std::max(nent, 1));
    const size_t oWh = carve(sizeof(double) * std::max(nent, 1));
    const size_t oWl = carve(sizeof(double) * std::max(nent, 1));
    const size_t oc = carve(sizeof(double) * d);
    const size_t ow = carve(sizeof(double) * d);
    const size_t ou = carve(sizeof(double));
    const size_t oFr = carve(sizeof(double2) * std::max(hp.tab_entries, 1));
    const size_t oFi = carve(p->two ? sizeof(double2) * std::max(hp.tab_entries, 1) : 0);
    const size_t oB = carve(sizeof(double) * 4);
    const size_t oS = carve(sizeof(int) * 4);
    const size_t oT = carve(sizeof(long long) * tabs.size());
    const size_t oScr = carve(sizeof(double) * 8);
    const size_t oCnt = carve(sizeof(unsigned long long) * 8);
    const size_t oSA = carve(sizeof(double) * (size_t)(L + 2) * (d + 1));
    const size_t oCm = carve(sizeof(double2) * hp.cm_hi.size());
    if (cudaMalloc(&p->dev_block, sz) != cudaSuccess) {
        cudaGetLastError();
        delete p;
        return SG_ENOMEM;
    }
    p->dev_bytes = sz;
    char *base = (char *)p->dev_block;
    DevPlan &dp = p->dp;
    memset(&dp, 0, sizeof dp);
    dp.d = d;
    dp.L = L;
    dp.kind = (int)f->kind;
    dp.nfront = hp.nfront;
    for (int l = 0; l < SG_MAX_L + 3; ++l) {
        dp.nl[l] = hp.nl[l];
        dp.entry_off[l] = hp.entry_off[l];
        dp.tab_off[l] = hp.tab_off[l];
    }
    for (int e = 0; e < SG_MAX_L + 2; ++e) dp.coef[e] = hp.coef[e];
    dp.M0 = hp.M0;
    dp.symmask = 0;
    for (int l = 2; l <= L + 1; ++l) {
        const int n = hp.nl[l], e0 = hp.entry_off[l];
        bool sym = n >= 2 && (n % 2 == 0 || hp.X[e0 + n / 2] == 0.5);
        for (int j = 0; sym && j < n / 2; ++j) {
            const int m = e0 + n - 1 - j;
            sym = (1.0 - hp.X[m] == hp.X[e0 + j]) && hp.Whi[m] == hp.Whi[e0 + j] && hp.Wlo[m] == hp.Wlo[e0 + j];
        }
        if (sym) dp.symmask |= 1 << l;
    }
    dp.X = (const double *)(base + oX);
    dp.Whi = (const double *)(base + oWh);
    dp.Wlo = (const double *)(base + oWl);
    dp.c = (const double *)(base + oc);
    dp.w = (const double *)(base + ow);
    dp.u = (const double *)(base + ou);
    dp.Fre = (double2 *)(base + oFr);
    dp.Fim = p->two ? (double2 *)(base + oFi) : nullptr;
    dp.sform = p->sform_dd ? 2 : p->sform ? 1 : 0;
    dp.base = (double *)(base + oB);
    dp.status = (int *)(base + oS);
    p->d_tabs = (long long *)(base + oT);
    p->d_scratch = (double *)(base + oScr);
    p->d_counter = (unsigned long long *)(base + oCnt);
    dp.SA = (double *)(base + oSA);
    dp.coefm = (const double2 *)(base + oCm);
    std::vector<double> wz(d, 0.0);
    std::vector<double2> cm(hp.cm_hi.size());
    for (size_t i = 0; i < cm.size(); ++i) cm[i] = make_double2(hp.cm_hi[i], hp.cm_lo[i]);
    bool ok = true;
    ok &= cudaMemcpy((void *)dp.X, hp.X.data(), sizeof(double) * nent, cudaMemcpyHostToDevice) == cudaSuccess;
    ok &= cudaMemcpy((void *)dp.Whi, hp.Whi.data(), sizeof(double) * nent, cudaMemcpyHostToDevice) == cudaSuccess;
    ok &= cudaMemcpy((void *)dp.Wlo, hp.Wlo.data(), sizeof(double) * nent, cudaMemcpyHostToDevice) == cudaSuccess;
    ok &= cudaMemcpy((void *)dp.c, f->c, sizeof(double) * d, cudaMemcpyHostToDevice) == cudaSuccess;
    ok &= cudaMemcpy((void *)dp.w, f->w ? f->w : wz.data(), sizeof(double) * d, cudaMemcpyHostToDevice) == cudaSuccess;
    ok &= cudaMemcpy((void *)dp.u, &f->u, sizeof(double), cudaMemcpyHostToDevice) == cudaSuccess;
    ok &= cudaMemcpy(p->d_tabs, tabs.data(), sizeof(long long) * tabs.size(), cudaMemcpyHostToDevice) == cudaSuccess;
    ok &= cudaMemset(dp.status, 0, sizeof(int) * 4) == cudaSuccess;
    ok &= cudaMemcpy((void *)dp.coefm, cm.data(), sizeof(double2) * cm.size(), cudaMemcpyHostToDevice) == cudaSuccess;
    if (!ok) {
        cudaGetLastError();
        cudaFree(p->dev_block);
        delete p;
        return SG_ECUDA;
    }
    rc = p->collapse ? SG_OK : setup_leaf1(p);
    if (rc) {
        cudaGetLastError();
        cudaFree(p->dev_block);
        delete p;
        return rc;
    }
    if (p->collapse) {
        // ---- collapse: workspace = the partial polynomials (re, im) of k_collapse_part ----
        p->collapse_blocks = (int)std::min<long long>(COLLAPSE_MAXB, (d + COLLAPSE_THREADS - 1) / COLLAPSE_THREADS);
        const size_t smem_part = (size_t)(p->cplx ? 4 : 2) * COLLAPSE_THREADS * (L + 1) * sizeof(double2);
        const size_t smem_fin = (size_t)(p->cplx ? 2 : 1) * COLLAPSE_THREADS * (L + 1) * sizeof(double2);
        cudaError_t e1, e2;
        if (p->cplx) {
            e1 = cudaFuncSetAttribute(k_collapse_part<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem_part);
            e2 = cudaFuncSetAttribute(k_collapse_final<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem_fin);
        } else {
            e1 = cudaFuncSetAttribute(k_collapse_part<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem_part);
            e2 = cudaFuncSetAttribute(k_collapse_final<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem_fin);
        }
        if (e1 != cudaSuccess || e2 != cudaSuccess) {
            cudaGetLastError();
            cudaFree(p->dev_block);
            delete p;
            return SG_ECUDA;
        }
        p->ws_part_off = 0;
        p->ws_need = align_up((size_t)2 * p->collapse_blocks * (L + 1) * sizeof(double2), 256);
        *out = p;
        return SG_OK;
    }
    // ---- workspace layout ----
    size_t ws = 0;
    const size_t rec = p->two ? 2 * sizeof(double2) : sizeof(double2);
    for (int par = 0; par < 2; ++par) {
        p->ws_front_off[par] = ws;
        ws = align_up(ws + (size_t)hp.ws_front_cap[par] * (rec + sizeof(uint32_t)) + 1024, 256);
    }
    p->ws_part_off = ws;
    ws = align_up(ws + sizeof(double2) * (size_t)std::max<int64_t>(hp.total_partials, 1), 256);
    p->ws_red_off = ws;
    ws = align_up(ws + sizeof(double2) * (size_t)((hp.total_partials + RED_CHUNK - 1) / RED_CHUNK + 1), 256);
    p->ws_need = ws;
    *out = p;
    return SG_OK;
}

extern "C" int sg_workspace_size(sg_plan_t p, size_t *bytes) {
    if (!p || !bytes) return SG_EINVAL;
    *bytes = p->ws_need;
    return SG_OK;
}

extern "C" int sg_set_workspace(sg_plan_t p, void *dev_ptr, size_t bytes) {
    if (!p || !dev_ptr) return SG_EINVAL;
    if (((uintptr_t)dev_ptr) % 256) return SG_EINVAL;
    if (bytes < p->ws_need) return SG_ENOMEM;
    p->ws = (char *)dev_ptr;
    p->ws_bytes = bytes;
    return SG_OK;
}

extern "C" int sg_update_integrand(sg_plan_t p, sg_stream_t s, const sg_integrand_desc *f) {
    if (!p) return SG_EINVAL;
    int rc = validate_desc(f, p->hp.d);
    if (rc) return rc;
    if ((int)f->kind != p->hp.kind) return SG_EINVAL;
    cudaStream_t st = (cudaStream_t)s;
    const size_t nb = sizeof(double) * p->hp.d;
    if (cudaMemcpyAsync((void *)p->dp.c, f->c, nb, cudaMemcpyDefault, st) != cudaSuccess) return SG_ECUDA;
    if (f->w && (f->kind == SG_F_PRODUCT_PEAK || f->kind == SG_F_GAUSSIAN))
        if (cudaMemcpyAsync((void *)p->dp.w, f->w, nb, cudaMemcpyDefault, st) != cudaSuccess) return SG_ECUDA;
    // u travels by value: staged through the plan's pinned-free path (a single 8-byte H2D copy)
    if (cudaMemcpyAsync((void *)p->dp.u, &f->u, sizeof(double), cudaMemcpyHostToDevice, st) != cudaSuccess)
        return SG_ECUDA;
    return SG_OK;
}

template <bool CPLX>
static const void *leaf1_kernel(int nj, bool smem) {
    if (nj == 3) return smem ? (const void *)k_leaf1<CPLX, 3, true> : (const void *)k_leaf1<CPLX, 3, false>;
    return smem ? (const void *)k_leaf1<CPLX, 2, true> : (const void *)k_leaf1<CPLX, 2, false>;
}

// Variant of k_leaf2 for this plan: NJ level-2 nodes, factor rows in smem or L1, midpoint index
// (center), symmetric pair (sym, oscillatory only), midpoint factor with zero low part (cz).
template <bool CPLX, bool SMEM>
static const void *leaf2_fn(int nj, bool center, bool sym, bool cz) {
    if (nj == 3 && center) {
        if (CPLX && sym) return cz ? (const void *)k_leaf2<CPLX, 3, SMEM, 1, true, true>
                                   : (const void *)k_leaf2<CPLX, 3, SMEM, 1, true, false>;
        return cz ? (const void *)k_leaf2<CPLX, 3, SMEM, 1, false, true> : (const void *)k_leaf2<CPLX, 3, SMEM, 1, false, false>;
    }
    if (nj == 3) return (const void *)k_leaf2<CPLX, 3, SMEM, -1>;
    if (CPLX && sym) return (const void *)k_leaf2<CPLX, 2, SMEM, -1, true>;
    return (const void *)k_leaf2<CPLX, 2, SMEM, -1>;
}
template <bool CPLX>
static const void *leaf2_kernel(int nj, bool smem, bool center, bool sym, bool cz) {
    return smem ? leaf2_fn<CPLX, true>(nj, center, sym, cz) : leaf2_fn<CPLX, false>(nj, center, sym, cz);
}

// Persistent geometry of the single-level last pass (k_leaf1, or the fused k_leaf2; once per plan).
static int setup_leaf1(sg_plan_s *p) {
    HostPlan &hp = p->hp;
    p->leaf1_t = -1;
    p->leaf2 = false;
    if (hp.nfront < 1 || p->sform) return SG_OK;
    const int t = hp.nfront, nj = hp.nl[2];
    if (hp.fuse) {
        p->leaf2 = true;
    } else {
        if (!p->leaf1) return SG_OK;
        if (t != hp.L - 1 || (nj != 2 && nj != 3)) return SG_OK;
    }
    const size_t smem = (size_t)hp.d * nj * sizeof(double2) * (p->cplx ? 2 : 1);
    p->leaf1_smem = smem <= 56 * 1024 ? smem : 0;
    const bool sm = p->leaf1_smem > 0;
    // midpoint node of the level-2 row (x = 1/2 exactly -> its oscillatory factor is exactly real)
    p->leaf2_center = (nj == 3 && hp.X[hp.entry_off[2] + 1] == 0.5);   // any kind
#ifdef LEAF2_NO_CENTER
    p->leaf2_center = false;
#endif
    const bool ct = p->leaf2_center;
    {
        // symmetric pair: x_0 + x_last == 1 and equal weights, exactly (NJ = 3 around the midpoint,
        // or NJ = 2 without one)
        const int e0 = hp.entry_off[2], e1 = e0 + nj - 1;
        p->leaf2_sym = (ct || nj == 2) && p->cplx && 1.0 - hp.X[e1] == hp.X[e0] && hp.Whi[e0] == hp.Whi[e1] &&
                       hp.Wlo[e0] == hp.Wlo[e1];
#ifdef LEAF2_NO_SYM
        p->leaf2_sym = false;
#endif
    }
    const bool sy = p->leaf2_sym;
    p->leaf2_cz = ct && hp.Wlo[hp.entry_off[2] + 1] == 0.0;
    const bool cz = p->leaf2_cz;
    const void *fn = p->leaf2 ? (p->cplx ? leaf2_kernel<true>(nj, sm, ct, sy, cz) : leaf2_kernel<false>(nj, sm, ct, sy, cz))
                              : (p->cplx ? leaf1_kernel<true>(nj, sm) : leaf1_kernel<false>(nj, sm));
    if (p->leaf1_smem > 48 * 1024 &&
        cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)p->leaf1_smem) != cudaSuccess)
        return SG_ECUDA;
    int per_sm = 0, dev = 0, sms = 0;
    if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, fn, PASS_THREADS, p->leaf1_smem) != cudaSuccess ||
        cudaGetDevice(&dev) != cudaSuccess ||
        cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess)
        return SG_ECUDA;
    const long long ntasks = hp.pass_ntasks[t];
    p->leaf1_grid = std::max<long long>(1, std::min<long long>((ntasks + WPB - 1) / WPB, (long long)sms * per_sm));
    hp.pass_blocks[t] = ntasks;   // partial slots: one per task (0 tasks -> no slot, no launch)
    int64_t poff = hp.root_blocks;
    for (int u = 1; u <= hp.nfront; ++u) {
        hp.pass_partial_off[u] = poff;
        poff += hp.pass_blocks[u];
    }
    hp.total_partials = poff;
    p->leaf1_t = t;
    return SG_OK;
}

template <bool CPLX>
static void launch_leaf2(sg_plan_s *p, const Leaf2Args &A, int nj, cudaStream_t st) {
    const unsigned grid = (unsigned)p->leaf1_grid;
    const size_t sm = p->leaf1_smem;
    const void *fn = leaf2_kernel<CPLX>(nj, sm > 0, p->leaf2_center, p->leaf2_sym, p->leaf2_cz);
    DevPlan dp = p->dp;
    Leaf2Args a = A;
    void *args[] = {&dp, &a};
    cudaLaunchKernel(fn, dim3(grid), dim3(PASS_THREADS), args, sm, st);
}

template <bool CPLX>
static void launch_leaf1(sg_plan_s *p, const PassArgs &A, int nj, cudaStream_t st) {
    const unsigned grid = (unsigned)p->leaf1_grid;
    const size_t sm = p->leaf1_smem;
    if (nj == 3) {
        if (sm) k_leaf1<CPLX, 3, true><<<grid, PASS_THREADS, sm, st>>>(p->dp, A);
        else k_leaf1<CPLX, 3, false><<<grid, PASS_THREADS, 0, st>>>(p->dp, A);
    } else {
        if (sm) k_leaf1<CPLX, 2, true><<<grid, PASS_THREADS, sm, st>>>(p->dp, A);
        else k_leaf1<CPLX, 2, false><<<grid, PASS_THREADS, 0, st>>>(p->dp, A);
    }
}

static void front_ptrs(sg_plan_s *p, int t, double2 *&re, double2 *&im, uint32_t *&meta) {
    const int par = t % 2;
    const int64_t cap = p->hp.ws_front_cap[par];
    char *b = p->ws + p->ws_front_off[par];
    re = (double2 *)b;
    im = p->two ? (double2 *)(b + sizeof(double2) * cap) : nullptr;
    meta = (uint32_t *)(b + (p->two ? 2 : 1) * sizeof(double2) * cap);
}

extern "C" int sg_integrate(sg_plan_t p, sg_stream_t s, double *out_dev) {
    if (!p || !out_dev) return SG_EINVAL;
    if (!p->ws) return SG_ENOWORKSPACE;
    cudaStream_t st = (cudaStream_t)s;
    const HostPlan &hp = p->hp;
    const DevPlan &dp = p->dp;
    double2 *partials = (double2 *)(p->ws + p->ws_part_off);
    if (cudaMemsetAsync(dp.status, 0, sizeof(int), st) != cudaSuccess) return SG_ECUDA;
    int evi = 0;
    auto mark = [&]() {
        if (p->prof && evi < (int)p->ev.size()) cudaEventRecord(p->ev[evi++], st);
    };
    mark();
    if (p->collapse) {
        const int L = hp.L;
        if (hp.tab_entries > 0) k_factor<<<(hp.tab_entries + 127) / 128, 128, 0, st>>>(dp);
        mark();
        k_base<<<1, 256, 0, st>>>(dp);
        mark();
        double2 *pre = (double2 *)(p->ws + p->ws_part_off);
        double2 *pim = pre + (size_t)p->collapse_blocks * (L + 1);
        const size_t smem_part = (size_t)(p->cplx ? 4 : 2) * COLLAPSE_THREADS * (L + 1) * sizeof(double2);
        const size_t smem_fin = (size_t)(p->cplx ? 2 : 1) * COLLAPSE_THREADS * (L + 1) * sizeof(double2);
        if (p->cplx) {
            k_collapse_part<true><<<p->collapse_blocks, COLLAPSE_THREADS, smem_part, st>>>(dp, pre, pim);
            mark();
            k_collapse_final<true><<<1, COLLAPSE_THREADS, smem_fin, st>>>(dp, pre, pim, p->collapse_blocks,
                                                                         p->collapse_emit ? 1 : 0, out_dev);
        } else {
            k_collapse_part<false><<<p->collapse_blocks, COLLAPSE_THREADS, smem_part, st>>>(dp, pre, pim);
            mark();
            k_collapse_final<false><<<1, COLLAPSE_THREADS, smem_fin, st>>>(dp, pre, pim, p->collapse_blocks,
                                                                          p->collapse_emit ? 1 : 0, out_dev);
        }
        mark();
        if (cudaGetLastError() != cudaSuccess) return SG_ECUDA;
        return SG_OK;
    }
    // K0
    if (hp.tab_entries > 0) {
        if (p->sform) {
            if (p->sform_dd) k_factor_s<true><<<(hp.tab_entries + 127) / 128, 128, 0, st>>>(dp);
            else k_factor_s<false><<<(hp.tab_entries + 127) / 128, 128, 0, st>>>(dp);
        } else {
            k_factor<<<(hp.tab_entries + 127) / 128, 128, 0, st>>>(dp);
            k_suffix_abs<<<hp.L, 256, 0, st>>>(dp);
        }
    }
    mark();
    if (p->sform) k_base_s<<<1, 256, 0, st>>>(dp);
    else k_base<<<1, 256, 0, st>>>(dp);
    mark();
    // root pass
    RootArgs R;
    memset(&R, 0, sizeof R);
    R.lo = hp.range_lo;
    R.hi = hp.range_hi;
    R.off1 = p->d_tabs + p->tab_off1;
    R.JS = p->d_tabs + p->tab_JS;
    if (hp.nfront >= 1) front_ptrs(p, 1, R.dst_re, R.dst_im, R.dst_meta);
    R.partials = partials;
    if (p->sform)
        (p->sform_dd ? k_root_s<true> : k_root_s<false>)<<<(unsigned)hp.root_blocks, 256, 0, st>>>(dp, R);
    else if (p->cplx)
        k_root<true><<<(unsigned)hp.root_blocks, 256, 0, st>>>(dp, R);
    else
        k_root<false><<<(unsigned)hp.root_blocks, 256, 0, st>>>(dp, R);
    mark();
    // level-synchronous passes
    for (int t = 1; t <= hp.nfront; ++t) {
        if (p->leaf2 && t == hp.nfront) {
            // fused last two levels: read the stored depth-(L-2) parents of excess L-2
            Leaf2Args B;
            memset(&B, 0, sizeof B);
            double2 *re, *im;
            uint32_t *meta;
            front_ptrs(p, t - 1, re, im, meta);
            B.src_re = re;
            B.src_im = im;
            B.base = hp.off[t - 1][(size_t)(hp.L - 2) * hp.d];
            B.Cmid = p->d_tabs + p->tab_CT[t - 1] + (size_t)(hp.L - 2) * hp.d;
            B.T2 = p->d_tabs + p->tab_TK;
            B.ntasks = hp.pass_ntasks[t];
            B.partials = partials + hp.pass_partial_off[t];
            B.counter = p->d_counter;
            if (cudaMemsetAsync(p->d_counter, 0, sizeof(unsigned long long), st) != cudaSuccess) return SG_ECUDA;
            if (B.ntasks > 0) {
                if (p->cplx) launch_leaf2<true>(p, B, hp.nl[2], st);
                else launch_leaf2<false>(p, B, hp.nl[2], st);
            }
            mark();
            continue;
        }
        PassArgs A;
        memset(&A, 0, sizeof A);
        A.nsrc = hp.total[t];
        A.ntasks = hp.pass_ntasks[t];
        A.nsplit = hp.pass_nsplit[t];
        A.t = t;
        double2 *re, *im;
        uint32_t *meta;
        front_ptrs(p, t, re, im, meta);
        A.src_re = re;
        A.src_im = im;
        A.src_meta = meta;
        const bool write = (t + 1 <= hp.nfront) && !(p->leaf2 && t + 1 == hp.nfront);
        if (write) front_ptrs(p, t + 1, A.dst_re, A.dst_im, A.dst_meta);
        A.offT = p->d_tabs + p->tab_offT[t];
        A.NT = p->d_tabs + p->tab_NT[t];
        A.CT = p->d_tabs + p->tab_CT[t];
        A.TB = write ? p->d_tabs + p->tab_TB[t] : nullptr;
        A.partials = partials + hp.pass_partial_off[t];
        A.counter = p->d_counter;
        if (t == p->leaf1_t && cudaMemsetAsync(p->d_counter, 0, sizeof(unsigned long long), st) != cudaSuccess)
            return SG_ECUDA;
        const unsigned grid = (unsigned)hp.pass_blocks[t];
        // single-level last pass (every source has excess L-1): specialised k_leaf1
        const int n2 = hp.nl[2];
        const bool single = !write && t == p->leaf1_t;
        if (p->sform) {
            if (p->sform_dd) {
                if (write) k_pass_s<true, true><<<grid, PASS_THREADS, 0, st>>>(dp, A);
                else k_pass_s<true, false><<<grid, PASS_THREADS, 0, st>>>(dp, A);
            } else {
                if (write) k_pass_s<false, true><<<grid, PASS_THREADS, 0, st>>>(dp, A);
                else k_pass_s<false, false><<<grid, PASS_THREADS, 0, st>>>(dp, A);
            }
        } else if (p->cplx) {
            if (write) k_pass<true, true><<<grid, PASS_THREADS, 0, st>>>(dp, A);
            else if (single) { if (A.ntasks > 0) launch_leaf1<true>(p, A, n2, st); }
            else k_leaf<true><<<grid, PASS_THREADS, 0, st>>>(dp, A);
        } else {
            if (write) k_pass<false, true><<<grid, PASS_THREADS, 0, st>>>(dp, A);
            else if (single) { if (A.ntasks > 0) launch_leaf1<false>(p, A, n2, st); }
            else k_leaf<false><<<grid, PASS_THREADS, 0, st>>>(dp, A);
        }
        mark();
    }
    {
        const long long nl1 = (hp.total_partials + RED_CHUNK - 1) / RED_CHUNK;
        double2 *l1 = (double2 *)(p->ws + p->ws_red_off);
        k_reduce_l1<<<(unsigned)nl1, 256, 0, st>>>(partials, hp.total_partials, l1);
        k_reduce<<<1, 1024, 0, st>>>(dp, l1, nl1, hp.include_root ? 1 : 0, out_dev);
    }
    mark();
    if (cudaGetLastError() != cudaSuccess) return SG_ECUDA;
    return SG_OK;
}

extern "C" int sg_finalize(sg_plan_t p, sg_stream_t s, const double *gathered_dev, int world,
                           double *result_dev) {
    if (!p || !gathered_dev || !result_dev || world < 1) return SG_EINVAL;
    k_finalize<<<1, 32, 0, (cudaStream_t)s>>>(gathered_dev, world, p->dp.status, result_dev);
    if (cudaGetLastError() != cudaSuccess) return SG_ECUDA;
    return SG_OK;
}

extern "C" int sg_integrate_host(sg_plan_t p, sg_stream_t s, double *result_host) {
    if (!p || !result_host) return SG_EINVAL;
    int rc = sg_integrate(p, s, p->d_scratch);
    if (rc) return rc;
    rc = sg_finalize(p, s, p->d_scratch, 1, p->d_scratch + 2);
    if (rc) return rc;
    if (cudaMemcpyAsync(result_host, p->d_scratch + 2, 2 * sizeof(double), cudaMemcpyDeviceToHost,
                        (cudaStream_t)s) != cudaSuccess)
        return SG_ECUDA;
    if (cudaStreamSynchronize((cudaStream_t)s) != cudaSuccess) return SG_ECUDA;
    if (!isfinite(result_host[0])) return SG_ENONFINITE;
    return SG_OK;
}

extern "C" int sg_status_word(sg_plan_t p, int *status) {
    if (!p || !status) return SG_EINVAL;
    int v = 0;
    if (cudaMemcpy(&v, p->dp.status, sizeof(int), cudaMemcpyDeviceToHost) != cudaSuccess) return SG_ECUDA;
    *status = v ? SG_ENONFINITE : SG_OK;
    return SG_OK;
}

extern "C" int sg_plan_points(sg_plan_t p, unsigned long long *shard_points,
                              unsigned long long *total_points) {
    if (!p) return SG_EINVAL;
    if (p->collapse) {   // the whole problem's n_d^q on rank 0 (not sharded)
        if (shard_points) *shard_points = p->collapse_emit ? p->hp.total_points : 0;
        if (total_points) *total_points = p->hp.total_points;
        return SG_OK;
    }
    if (shard_points) *shard_points = p->hp.shard_points;
    if (total_points) *total_points = p->hp.total_points;
    return SG_OK;
}

extern "C" int sg_plan_range(sg_plan_t p, long long *lo, long long *hi, long long *n_depth1) {
    if (!p) return SG_EINVAL;
    if (lo) *lo = p->hp.range_lo;
    if (hi) *hi = p->hp.range_hi;
    if (n_depth1) *n_depth1 = (long long)p->hp.d * p->hp.M0;
    return SG_OK;
}

extern "C" int sg_plan_passes(sg_plan_t p, int *npass, unsigned long long *terms,
                              unsigned long long *written) {
    if (!p || !npass) return SG_EINVAL;
    const int n = p->collapse ? 0 : p->hp.nfront + 1;   // the collapse runs no tree passes
    if ((terms || written) && *npass < n) {
        *npass = n;
        return SG_EINVAL;
    }
    *npass = n;
    for (int i = 0; i < n; ++i) {
        if (terms) terms[i] = p->hp.pass_terms[i];
        if (written) written[i] = p->hp.pass_written[i];
    }
    return SG_OK;
}

// FP64 instruction mix per leaf of the last pass's kernel variant (counted from the leaf helpers
// above: leaf1_term real 4 DFMA + 3 DADD, complex 8 + 6; leaf_real_factor_term 4 + 3, or 3 + 3
// with CZ; leaf_sym_pair_terms 8 + 10 for its two leaves).
extern "C" int sg_plan_leaf_work(sg_plan_t p, double *dfma_per_point, double *dadd_per_point) {
    if (!p || !dfma_per_point || !dadd_per_point) return SG_EINVAL;
    // biased grid accumulator (leaf_term): generic real 4 DFMA + 2 DADD, oscillatory 8 + 4;
    // symmetric pair 8 + 8 for two points; real midpoint factor 3 (CZ) / 4 DFMA + 2 DADD
    double f = p->cplx ? 8.0 : 4.0, a = p->cplx ? 4.0 : 2.0;
    if (p->leaf2 && p->leaf2_sym && !p->leaf2_center) {   // NJ = 2 symmetric pair
        f = 8.0 / 2.0;
        a = 8.0 / 2.0;
    } else if (p->leaf2 && p->leaf2_center) {
        const double cf = p->leaf2_cz ? 3.0 : 4.0, ca = 2.0;
        if (p->leaf2_sym) {
            f = (8.0 + cf) / 3.0;
            a = (8.0 + ca) / 3.0;
        } else {
            f = (2.0 * f + cf) / 3.0;
            a = (2.0 * a + ca) / 3.0;
        }
    }
    *dfma_per_point = f;
    *dadd_per_point = a;
    return SG_OK;
}

extern "C" int sg_debug_tables(sg_plan_t p, double *table_host, size_t table_doubles, double *base_host) {
    if (!p) return SG_EINVAL;
    const size_t per = p->two ? 4 : 2, n = (size_t)p->hp.tab_entries;
    if (table_host) {
        if (table_doubles < n * per) return SG_EINVAL;
        std::vector<double2> re(n), im(p->two ? n : 0);
        if (cudaMemcpy(re.data(), p->dp.Fre, sizeof(double2) * n, cudaMemcpyDeviceToHost) != cudaSuccess)
            return SG_ECUDA;
        if (p->two && cudaMemcpy(im.data(), p->dp.Fim, sizeof(double2) * n, cudaMemcpyDeviceToHost) != cudaSuccess)
            return SG_ECUDA;
        for (size_t i = 0; i < n; ++i) {
            table_host[i * per + 0] = re[i].x;
            table_host[i * per + 1] = re[i].y;
            if (p->two) {
                table_host[i * per + 2] = im[i].x;
                table_host[i * per + 3] = im[i].y;
            }
        }
    }
    if (base_host)
        if (cudaMemcpy(base_host, p->dp.base, 4 * sizeof(double), cudaMemcpyDeviceToHost) != cudaSuccess)
            return SG_ECUDA;
    return SG_OK;
}

extern "C" int sg_plan_query(int d, int q, sg_rule rule, sg_kind kind, const sg_options *opt,
                             unsigned long long *shard_points, unsigned long long *total_points,
                             long long *range_lo, long long *range_hi, int *n_passes) {
    if (d < 1 || q < d) return SG_EINVAL;
    sg_options o = {SG_FORM_COMBINATION, SG_ARITH_FACTOR_DD, 0, 1, 0, -1};
    if (opt) o = *opt;
    if (o.arith != SG_ARITH_FACTOR_DD && o.arith != SG_ARITH_SFORM_FP64 && o.arith != SG_ARITH_SFORM_DD)
        return SG_EINVAL;
    HostPlan hp;
    int rc = host_plan_build(hp, d, q - d, (int)rule, (int)kind, (int)o.form, (int)o.merge, o.rank, o.world,
                             o.range_lo, o.range_hi);
    if (rc) return rc;
    if (shard_points) *shard_points = hp.shard_points;
    if (total_points) *total_points = hp.total_points;
    if (range_lo) *range_lo = hp.range_lo;
    if (range_hi) *range_hi = hp.range_hi;
    if (n_passes) *n_passes = hp.nfront + 1;
    return SG_OK;
}

extern "C" int sg_unrank(int d, int q, sg_rule rule, sg_kind kind, const sg_options *opt,
                         unsigned long long index, int *t, int *k, int *l, int *j, double *coef) {
    if (d < 1 || q < d || !t || !k || !l || !j || !coef) return SG_EINVAL;
    sg_options o = {SG_FORM_COMBINATION, SG_ARITH_FACTOR_DD, 0, 1, 0, -1};
    if (opt) o = *opt;
    HostPlan hp;
    int rc = host_plan_build(hp, d, q - d, (int)rule, (int)kind, (int)o.form, (int)o.merge, o.rank, o.world,
                             o.range_lo, o.range_hi, 0);
    if (rc) return rc;
    return host_unrank(hp, index, t, k, l, j, coef);
}

extern "C" int sg_rule_table(sg_rule rule, int level, double *x, double *w) {
    if (!x || !w || level < 1) return SG_EINVAL;
    if (rule != SG_RULE_CLENSHAW_CURTIS && rule != SG_RULE_GAUSS_LEGENDRE && rule != SG_RULE_TRAPEZOIDAL &&
        rule != SG_RULE_GAUSS_PATTERSON)
        return SG_EINVAL;
    int n = host_rule((int)rule, level, x, w);
    return n < 0 ? SG_EUNSUPPORTED : n;
}

extern "C" int sg_profile_enable(sg_plan_t p, int enable) {
    if (!p) return SG_EINVAL;
    if (enable && p->ev.empty()) {
        p->ev.resize(5 + p->hp.nfront);
        for (auto &e : p->ev)
            if (cudaEventCreate(&e) != cudaSuccess) return SG_ECUDA;
    }
    p->prof = enable != 0;
    return SG_OK;
}

extern "C" int sg_profile_read(sg_plan_t p, float *ms, int *n) {
    if (!p || !n) return SG_EINVAL;
    // launches: tree [K0 factor, K0 base, root, pass 1..nfront, reduce];
    //           collapse [K0 factor, K0 base, k_collapse_part, k_collapse_final]
    const int nl = p->collapse ? 4 : 4 + p->hp.nfront;
    if (!ms) {
        *n = nl;
        return SG_OK;
    }
    if (*n < nl || p->ev.empty()) return SG_EINVAL;
    if (cudaEventSynchronize(p->ev[nl]) != cudaSuccess) return SG_ECUDA;
    for (int i = 0; i < nl; ++i)
        if (cudaEventElapsedTime(&ms[i], p->ev[i], p->ev[i + 1]) != cudaSuccess) return SG_ECUDA;
    *n = nl;
    return SG_OK;
}

extern "C" int sg_destroy(sg_plan_t p) {
    if (!p) return SG_EINVAL;
    for (auto &e : p->ev) cudaEventDestroy(e);
    if (p->dev_block) cudaFree(p->dev_block);
    delete p;
    return SG_OK;
}
