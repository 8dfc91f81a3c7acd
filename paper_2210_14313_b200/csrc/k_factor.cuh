// k_factor.cuh — K0: per-(level, coordinate, node) factor tables, the base value and the suffix bounds of |F|
// (included once, by sg_kernels.cu, after the shared definitions it uses)
#pragma once

// ---------------------------------------------------------------------------------------------
// K0: factor table and base
// ---------------------------------------------------------------------------------------------
__device__ __forceinline__ bool dd_finite(dd a) { return isfinite(a.hi) && isfinite(a.lo); }

struct FactorOut {
    int l, k, j;   // level, coordinate, node of the entry
    dd Fr, Fi;     // its factor w E (imaginary part: oscillatory kind)
};

template <int KIND>
__device__ __forceinline__ void factor_entry(const DevPlan &P, int idx, FactorOut *outp = nullptr) {
    const int n_ent = P.tab_off[P.L + 2];
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
    switch (KIND) {
    case SG_F_EXP_LINEAR:
        Er = dd_exp_ool(dd_mul_d(xm, ck));
        break;
    case SG_F_OSCILLATORY: {
        // sincos of |a| with the sign applied afterwards: nodes placed symmetrically about 1/2 get
        // exactly conjugate factors (used by k_leaf2's symmetric-pair path)
        dd a = dd_mul_d(xm, ck), s, co;
        const bool neg = a.hi < 0.0;
        dd_sincos_ool(neg ? dd_neg(a) : a, s, co);
        Er = co;
        Ei = neg ? dd_neg(s) : s;
        break;
    }
    case SG_F_GAUSSIAN: {
        // -c^2 ((x-w)^2 - (1/2-w)^2) = -c^2 (x - 1/2)(x + 1/2 - 2w)
        const double wk = P.w[k];
        dd xp = dd_add(dd_from_sum(x, 0.5), dd{-2.0 * wk, 0.0});
        dd arg = dd_mul(dd_mul(xm, xp), dd_from_prod(ck, ck));
        Er = dd_exp_ool(dd_neg(arg));
        break;
    }
    case SG_F_PRODUCT_PEAK: {
        // phi(x)/phi(1/2) = (c^-2 + (1/2-w)^2) / (c^-2 + (x-w)^2)
        const double wk = P.w[k];
        dd ci2 = dd_div_ool(dd{1.0, 0.0}, dd_from_prod(ck, ck));
        dd a = dd_from_sum(x, -wk), bm = dd_from_sum(0.5, -wk);
        Er = dd_div_ool(dd_add(ci2, dd_mul(bm, bm)), dd_add(ci2, dd_mul(a, a)));
        break;
    }
    }
    dd Fr = dd_mul(wt, Er), Fi = {0.0, 0.0};
    P.Fre[idx] = make_double2(Fr.hi, Fr.lo);
    bool ok = dd_finite(Fr);
    if (KIND == SG_F_OSCILLATORY) {
        Fi = dd_mul(wt, Ei);
        P.Fim[idx] = make_double2(Fi.hi, Fi.lo);
        ok = ok && dd_finite(Fi);
    }
    if (!ok) atomicOr(P.status, 1);
    if (outp) *outp = FactorOut{l, k, j, Fr, Fi};
}

// per-coordinate bound b_k >= max over x in [0,1] of |E_k(x)| (|Re| + |Im| for the oscillatory kind),
// evaluated in FP64 with a relative margin of 2^-40 over the library exp's error: the analytic
// suffix bounds SA (k_head) use it instead of summing the table's |F|
template <int KIND>
__device__ __forceinline__ double coord_bound(const DevPlan &P, int k) {
    const double ck = P.c[k];
    switch (KIND) {
    case SG_F_EXP_LINEAR: return exp(0.5 * fabs(ck)) * (1.0 + 0x1p-40);
    case SG_F_OSCILLATORY: return 1.4142135623730951 * (1.0 + 0x1p-40);
    case SG_F_GAUSSIAN: {
        // exp(-c^2 ((x - w)^2 - (1/2 - w)^2)) is largest where (x - w)^2 is smallest on [0, 1]
        const double wk = P.w[k], dist = wk < 0.0 ? -wk : (wk > 1.0 ? wk - 1.0 : 0.0), bm = 0.5 - wk;
        return exp(ck * ck * (bm * bm - dist * dist)) * (1.0 + 0x1p-40);
    }
    case SG_F_PRODUCT_PEAK: {
        const double wk = P.w[k], dist = wk < 0.0 ? -wk : (wk > 1.0 ? wk - 1.0 : 0.0), bm = 0.5 - wk;
        const double ci2 = 1.0 / (ck * ck);
        return (ci2 + bm * bm) / (ci2 + dist * dist) * (1.0 + 0x1p-40);
    }
    }
    return 1.0;
}

// base value B (256-thread CTA): fixed-order strided partials, then a fixed CTA tree (sum; product
// for the peak kind)
template <int KIND>
__device__ __forceinline__ void base_body(const DevPlan &P) {
    const bool prod = (KIND == SG_F_PRODUCT_PEAK);
    dd acc = prod ? dd{1.0, 0.0} : dd{0.0, 0.0};
    for (int k = threadIdx.x; k < P.d; k += blockDim.x) {
        const double ck = P.c[k];
        switch (KIND) {
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
            dd ci2 = dd_div_ool(dd{1.0, 0.0}, dd_from_prod(ck, ck));
            acc = dd_mul(acc, dd_div_ool(dd{1.0, 0.0}, dd_add(ci2, dd_mul(bm, bm))));
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
        switch (KIND) {
        case SG_F_EXP_LINEAR: Br = dd_exp_ool(s); break;
        case SG_F_GAUSSIAN: Br = dd_exp_ool(dd_neg(s)); break;
        case SG_F_PRODUCT_PEAK: Br = s; break;
        case SG_F_OSCILLATORY: {
            const double u = P.u[0];
            dd th = dd_add(dd_from_prod(DD_2PI_0, u), dd_from_prod(DD_2PI_1, u));
            th = dd_add(th, dd{DD_2PI_2 * u, 0.0});
            th = dd_add(th, s);
            dd sn, cs;
            dd_sincos_ool(th, sn, cs);
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

// K0 in one launch: blocks 0 .. nfb-1 fill the factor table (one entry per thread), block nfb computes
// the base value (independent of the table; base_body needs a 256-thread block).
#define K0_THREADS 256
// KIND: the integrand kind (one instantiation each: the others' dd exp / sincos / division code would
// only cost instruction fetches in this latency-bound launch)
template <int KIND>
__global__ void __launch_bounds__(K0_THREADS) k_factor_base(const DevPlan P, int nfb) {
    if ((int)blockIdx.x == nfb) base_body<KIND>(P);
    else factor_entry<KIND>(P, blockIdx.x * K0_THREADS + threadIdx.x);
}

// SA[l][k] = sum_{k' >= k} sum_j (|Fre[l][k'][j].hi| + |Fim[l][k'][j].hi|): bound used by the leaf
// kernels' grid accumulators.  One CTA per level: chunked row sums, a parallel (Hillis-Steele)
// suffix scan over the chunk sums, then each thread writes the suffix values of its chunk.  SA is
// only an upper bound for the grid choice (used with a 1 + 2^-20 margin), so the summation order is
// free; it is fixed, so SA is deterministic.  (Tried: the same scan in K0's last block (atomic
// ticket) to save the launch: 21 us slower on config 4 — one 256-thread CTA walking the levels in
// turn is latency-bound; reverted.)
#define SUFFIX_THREADS 1024
__global__ void __launch_bounds__(SUFFIX_THREADS) k_suffix_abs(const DevPlan P) {
    const int l = 2 + blockIdx.x;
    if (l > P.L + 1) return;
    const int d = P.d, n = P.nl[l];
    const double2 *Fr = P.Fre + P.tab_off[l];
    const double2 *Fi = P.kind == SG_F_OSCILLATORY ? P.Fim + P.tab_off[l] : nullptr;
    const int chunk = (d + SUFFIX_THREADS - 1) / SUFFIX_THREADS;
    const int k0 = min(d, (int)threadIdx.x * chunk), k1 = min(d, k0 + chunk);
    auto row = [&](int k) {
        double r0 = 0.0, r1 = 0.0;
        const double2 *fr = Fr + (long long)k * n;
        const double2 *fi = Fi ? Fi + (long long)k * n : nullptr;
#pragma unroll 4
        for (int j = 0; j < n; ++j) {
            r0 += fabs(__ldg(fr + j).x);
            if (fi) r1 += fabs(__ldg(fi + j).x);
        }
        return r0 + r1;
    };
    double cs = 0.0;
    for (int k = k0; k < k1; ++k) cs += row(k);
    __shared__ double suf[SUFFIX_THREADS + 1];
    suf[threadIdx.x] = cs;
    if (threadIdx.x == 0) suf[SUFFIX_THREADS] = 0.0;
    __syncthreads();
    for (int off = 1; off < SUFFIX_THREADS; off <<= 1) {   // suf[i] = sum of chunks i.. end
        const double t = (threadIdx.x + off < SUFFIX_THREADS) ? suf[threadIdx.x + off] : 0.0;
        __syncthreads();
        suf[threadIdx.x] += t;
        __syncthreads();
    }
    double sacc = suf[threadIdx.x + 1];   // sum of the chunks after this thread's chunk
    if (threadIdx.x == 0) P.SA[(long long)l * (d + 1) + d] = 0.0;
    for (int k = k1 - 1; k >= k0; --k) {
        sacc += row(k);
        P.SA[(long long)l * (d + 1) + k] = sacc;
    }
}

// ---------------------------------------------------------------------------------------------
// k_head: the head of a tree step in ONE launch, no grid barrier — K0's factor entries, the base B
// (every block computes it redundantly from the d coefficients: the same fixed-order arithmetic, so
// the same bits; block 0 stores it), the root pass for the block's own entries (the depth-1 point of
// entry (l, k, j) is rank r1 = k M0 + sum_{l'<l} n_l' + j; its factor is the thread's own, so no
// cross-block dependency), and, in block 0, the analytic suffix bounds SA[l][k] = W_l sum_{k'>=k}
// b_k' (W_l = sum_j |w_j^l|, b_k = coord_bound) — upper bounds of the table sums k_suffix_abs takes.
// Replaces k_factor_base + k_suffix_abs + k_root (three graph nodes) for d <= HEAD_MAX_D, where the
// redundant per-block base loop (d / 256 coordinates per thread) stays short.  Root partial slot =
// the block (plan.cpp sizes root_blocks to the K0 grid).
// CTA = K0_THREADS entry threads (warps 0-7, one factor entry each) + one helper warp.  B's
// coordinate sum and CTA tree come first; then the helper's lane 0 evaluates B's dd exp / sincos
// WHILE the entry threads evaluate their entries' (the two transcendental chains overlap instead of
// following each other: configs 1-2 0.036 -> 0.032 ms, 0.096 -> 0.094 ms) and exits; the entry
// threads then run the root pass, the block partial and (block 0) the suffix bounds, synchronised
// by named barrier 1 over the K0_THREADS entry threads.  (The suffix bounds by the helper warp
// alone, beside the root pass, were slower for d = 1000: 32 coordinates per lane.)
// ---------------------------------------------------------------------------------------------
#define HEAD_MAX_D 2048
#define HEAD_THREADS (K0_THREADS + 32)

template <int KIND>
__global__ void __launch_bounds__(HEAD_THREADS) k_head(const DevPlan P, const RootArgs R) {
    constexpr bool CPLX = (KIND == SG_F_OSCILLATORY);
    const bool helper = threadIdx.x >= K0_THREADS;
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    const int idx = blockIdx.x * K0_THREADS + threadIdx.x;
    __shared__ double2 bsm[2];
    __shared__ double2 sm[K0_THREADS];
    // (1) B's coordinate sum (product for the peak kind): base_body's strided partials and CTA tree
    constexpr bool prod = (KIND == SG_F_PRODUCT_PEAK);
    if (!helper) {
        dd acc = prod ? dd{1.0, 0.0} : dd{0.0, 0.0};
        for (int k = threadIdx.x; k < P.d; k += K0_THREADS) {
            const double ck = P.c[k];
            switch (KIND) {
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
                dd ci2 = dd_div_ool(dd{1.0, 0.0}, dd_from_prod(ck, ck));
                acc = dd_mul(acc, dd_div_ool(dd{1.0, 0.0}, dd_add(ci2, dd_mul(bm, bm))));
                break;
            }
            }
        }
        sm[threadIdx.x] = make_double2(acc.hi, acc.lo);
    }
    __syncthreads();
    for (int s2 = K0_THREADS / 2; s2 > 0; s2 >>= 1) {
        if (threadIdx.x < s2) {
            dd a = {sm[threadIdx.x].x, sm[threadIdx.x].y}, b = {sm[threadIdx.x + s2].x, sm[threadIdx.x + s2].y};
            dd r = prod ? dd_mul(a, b) : dd_add(a, b);
            sm[threadIdx.x] = make_double2(r.hi, r.lo);
        }
        __syncthreads();
    }
    // (2) helper lane 0: B from the sum; entry threads: their factor entries (concurrently)
    FactorOut fo;
    fo.l = -1;
    if (helper) {
        if (threadIdx.x == K0_THREADS) {
            dd sv = {sm[0].x, sm[0].y};
            dd Br = sv, Bi = {0.0, 0.0};
            switch (KIND) {
            case SG_F_EXP_LINEAR: Br = dd_exp_ool(sv); break;
            case SG_F_GAUSSIAN: Br = dd_exp_ool(dd_neg(sv)); break;
            case SG_F_PRODUCT_PEAK: Br = sv; break;
            case SG_F_OSCILLATORY: {
                const double u = P.u[0];
                dd th = dd_add(dd_from_prod(DD_2PI_0, u), dd_from_prod(DD_2PI_1, u));
                th = dd_add(th, dd{DD_2PI_2 * u, 0.0});
                th = dd_add(th, sv);
                dd sn, cs;
                dd_sincos_ool(th, sn, cs);
                Br = cs;
                Bi = sn;
                break;
            }
            }
            bsm[0] = make_double2(Br.hi, Br.lo);
            bsm[1] = make_double2(Bi.hi, Bi.lo);
            if (blockIdx.x == 0) {
                P.base[0] = Br.hi;
                P.base[1] = Br.lo;
                P.base[2] = Bi.hi;
                P.base[3] = Bi.lo;
                if (!dd_finite(Br) || !dd_finite(Bi)) atomicOr(P.status, 1);
            }
        }
    } else {
        factor_entry<KIND>(P, idx, &fo);
    }
    __syncthreads();
    if (helper) return;   // no further barrier 0: the entry threads use named barrier 1
    // (3a) root pass for this thread's entry (k_root's arithmetic)
    dd tot = {0.0, 0.0};
    if (fo.l >= 2) {
        long long r1 = (long long)fo.k * P.M0 + fo.j;
        for (int l = 2; l < fo.l; ++l) r1 += P.nl[l];
        if (r1 >= R.lo && r1 < R.hi) {
            const dd Br = {bsm[0].x, bsm[0].y};
            dd cr, ci = {0.0, 0.0};
            if (CPLX) {
                const dd Bi = {bsm[1].x, bsm[1].y};
                cdd ch = cdd_mul(cdd{Br, Bi}, cdd{fo.Fr, fo.Fi});
                cr = ch.re;
                ci = ch.im;
            } else {
                cr = dd_mul(Br, fo.Fr);
            }
            const int b1 = fo.l - 1, k1 = fo.k;
            tot = coef_mul(P, cr, 1, b1);
            if (P.nfront >= 1 && b1 <= P.L - 1 && k1 <= P.d - 2) {
                const long long seg = (long long)b1 * P.d + k1;
                const long long o = R.off1[seg] + fo.j - R.JS[seg];
                SG_DST(R, dst_re, o) = make_double2(cr.hi, cr.lo);
                if (CPLX) SG_DST(R, dst_im, o) = make_double2(ci.hi, ci.lo);
                SG_DST(R, dst_meta, o) = ((uint32_t)b1 << SG_META_KBITS) | (uint32_t)k1;
            }
        }
    }
    // block partial: block_reduce_dd's arithmetic over the entry warps, synchronised by named
    // barrier 1 (K0_THREADS threads; the helper warp does not take part)
    dd v = warp_reduce_dd(tot);
    __shared__ double2 rsm[K0_THREADS / 32];
    if (lane == 0) rsm[wid] = make_double2(v.hi, v.lo);
    asm volatile("bar.sync 1, %0;" ::"r"(K0_THREADS) : "memory");
    if (threadIdx.x == 0) {
        dd sblk = {0.0, 0.0};
        for (int i = 0; i < K0_THREADS / 32; ++i) sblk = dd_add(sblk, dd{rsm[i].x, rsm[i].y});
        SG_PART(R.partials, blockIdx.x) = make_double2(sblk.hi, sblk.lo);
    }
    // block 0: analytic suffix bounds of every level (chunk sums, a Hillis-Steele suffix scan over
    // the K0_THREADS chunks, then each thread writes its chunk's suffix values)
    if (blockIdx.x == 0) {
        const int d = P.d, chunk = (d + K0_THREADS - 1) / K0_THREADS;   // <= HEAD_MAX_D / K0_THREADS
        const int k0 = min(d, (int)threadIdx.x * chunk), k1 = min(d, k0 + chunk);
        double bk[HEAD_MAX_D / K0_THREADS];
        double cs = 0.0;
#pragma unroll
        for (int c = 0; c < HEAD_MAX_D / K0_THREADS; ++c) {
            bk[c] = (k0 + c < k1) ? coord_bound<KIND>(P, k0 + c) : 0.0;
            cs += bk[c];
        }
        __shared__ double suf[K0_THREADS + 1];
        suf[threadIdx.x] = cs;
        if (threadIdx.x == 0) suf[K0_THREADS] = 0.0;
        asm volatile("bar.sync 1, %0;" ::"r"(K0_THREADS) : "memory");
        for (int off = 1; off < K0_THREADS; off <<= 1) {   // suf[i] = sum of chunks i.. end
            const double t = (threadIdx.x + off < K0_THREADS) ? suf[threadIdx.x + off] : 0.0;
            asm volatile("bar.sync 1, %0;" ::"r"(K0_THREADS) : "memory");
            suf[threadIdx.x] += t;
            asm volatile("bar.sync 1, %0;" ::"r"(K0_THREADS) : "memory");
        }
        double sacc = suf[threadIdx.x + 1];
        double sk[HEAD_MAX_D / K0_THREADS];
#pragma unroll
        for (int c = HEAD_MAX_D / K0_THREADS - 1; c >= 0; --c) {
            sacc += bk[c];
            sk[c] = sacc;
        }
        for (int l = 2; l <= P.L + 1; ++l) {
            const double wl = P.wabs[l] * (1.0 + 0x1p-40);
            if (threadIdx.x == 0) P.SA[(long long)l * (d + 1) + d] = 0.0;
#pragma unroll
            for (int c = 0; c < HEAD_MAX_D / K0_THREADS; ++c)
                if (k0 + c < k1) P.SA[(long long)l * (d + 1) + k0 + c] = wl * sk[c];
        }
    }
}
