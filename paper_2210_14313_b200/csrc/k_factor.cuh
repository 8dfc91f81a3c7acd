// k_factor.cuh — K0: per-(level, coordinate, node) factor tables, the base value and the suffix bounds of |F|
// (included once, by sg_kernels.cu, after the shared definitions it uses)
#pragma once

// ---------------------------------------------------------------------------------------------
// K0: factor table and base
// ---------------------------------------------------------------------------------------------
__device__ __forceinline__ bool dd_finite(dd a) { return isfinite(a.hi) && isfinite(a.lo); }

__device__ __forceinline__ void factor_entry(const DevPlan &P, int idx) {
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

// base value B (256-thread CTA): fixed-order strided partials, then a fixed CTA tree (sum; product
// for the peak kind)
__device__ __forceinline__ void base_body(const DevPlan &P) {
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

// K0 in one launch: blocks 0 .. nfb-1 fill the factor table (one entry per thread), block nfb computes
// the base value (independent of the table; base_body needs a 256-thread block).
#define K0_THREADS 256
__global__ void __launch_bounds__(K0_THREADS) k_factor_base(const DevPlan P, int nfb) {
    if ((int)blockIdx.x == nfb) base_body(P);
    else factor_entry(P, blockIdx.x * K0_THREADS + threadIdx.x);
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
