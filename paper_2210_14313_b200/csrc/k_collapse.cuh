// k_collapse.cuh — separable collapse (SG_METHOD_COLLAPSE): per-coordinate polynomials in the level budget
// (included once, by sg_kernels.cu, after the shared definitions it uses)
#pragma once

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
        const int st = *P.status || !dd_finite(a);
        if (st) a = dd{nan(""), nan("")};
        out[0] = a.hi;
        out[1] = a.lo;
        step_close_status(P, st);
    }
}

