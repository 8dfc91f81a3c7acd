// k_sform.cuh — s-form passes: partial sums of the argument, outer function per point (FP64 ablation and dd)
// (included once, by sg_kernels.cu, after the shared definitions it uses)
#pragma once

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
__device__ __forceinline__ void factor_s_entry(const DevPlan &P, int idx) {
    const int n_ent = P.tab_off[P.L + 2];
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
__device__ __forceinline__ void base_s_body(const DevPlan &P) {
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

// K0 of the s-form in one launch (block nfb: the base sum S; see k_factor_base)
template <bool DDS>
__global__ void __launch_bounds__(K0_THREADS) k_factor_base_s(const DevPlan P, int nfb) {
    if ((int)blockIdx.x == nfb) base_s_body(P);
    else factor_s_entry<DDS>(P, blockIdx.x * K0_THREADS + threadIdx.x);
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
            SG_DST(R, dst_re, o) = wv;
            SG_DST(R, dst_im, o) = av;
            SG_DST(R, dst_meta, o) = ((uint32_t)b1 << SG_META_KBITS) | (uint32_t)k1;
        }
    }
    dd s = block_reduce_dd<8>(tot);
    if (threadIdx.x == 0) SG_PART(R.partials, blockIdx.x) = make_double2(s.hi, s.lo);
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
            const uint32_t m = SG_SRC(A, src_meta, g);
            b = (int)(m >> SG_META_KBITS);
            k = (int)(m & META_KMASK);
            const double2 v = SG_SRC(A, src_re, g), dv = SG_SRC(A, src_im, g);
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
        const dd y0 = DDS ? dd_add(S, delta) : dd{0.0, 0.0};   // the lane's argument before its child
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
                    // dd: the point's argument (S + delta) + a (one dd add; the child's own delta
                    // is only formed when it is stored); FP64 ablation: S + (delta + a)
                    const dd dl = DDS ? ((WRITE && wk) ? dd_add(delta, dd{av.x, av.y}) : dd{0.0, 0.0})
                                      : dd{delta.hi + av.x, 0.0};
                    const dd Wc = dd_mul(W, dd{wv.x, wv.y});
                    dd gv = {0.0, 0.0};
                    if (kv) gv = sform_value<DDS>(P, DDS ? dd_add(y0, dd{av.x, av.y}) : dd{S.hi + dl.hi, 0.0});
                    double p, e;
                    dd_mul_pe(Wc, gv, p, e);
                    acc_add(ah, al, p, e);
                    if (WRITE && wk) {
                        const long long o = tb + (long long)j * Nseg;
                        SG_DST(A, dst_re, o) = make_double2(Wc.hi, Wc.lo);
                        SG_DST(A, dst_im, o) = make_double2(dl.hi, dl.lo);
                        SG_DST(A, dst_meta, o) = ((uint32_t)bp << SG_META_KBITS) | (uint32_t)kp;
                    }
                }
            }
            if (lv) tot = dd_add(tot, dd_mul_d(dd_norm(ah, al), P.coef[bp]));
        }
    }
    dd s = block_reduce_dd<WPB>(tot);
    if (threadIdx.x == 0) SG_PART(A.partials, blockIdx.x) = make_double2(s.hi, s.lo);
}

