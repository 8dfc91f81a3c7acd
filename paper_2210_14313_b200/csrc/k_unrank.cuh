// k_unrank.cuh — K1 on the device: flat point index -> (multi-index, tensor point, coefficient), and
// the point's term evaluated on its own (sg_eval_points).
// (included once, by sg_kernels.cu, after the shared definitions it uses)
#pragma once

// Tables (plan-owned, built lazily by sg_eval_points):
//   Sub[b * (d+1) + (k+1)]  points (nonzero coefficient) in the subtree of a node of excess b whose
//                           last active coordinate is k (k = -1: the root), the node included;
//   SG[b * (d+1) + k]       sum_{k' >= k} sum_{l'} n_{l'} Sub[b + l' - 1][k'] (children blocks after
//                           coordinate k-1 of a node of excess b; SG[b][d] = 0);
//   D1[i]                   points in the depth-1 subtrees r1 = lo .. lo+i-1 of the shard (prefix).
// The canonical order is host_unrank's (plan.cpp): the root (if in the shard and counted), then the
// depth-1 subtrees in r1 order, each in preorder with children ordered by (k', l', j').
struct UnrankTabs {
    const unsigned long long *Sub, *SG, *D1;
    long long lo, n1;        // shard depth-1 range [lo, lo + n1)
    int include_root, merge;
    unsigned long long shard_points;
};

// Returns depth t (>= 0) and writes the active triples; -1 for an index outside the shard.
__device__ int unrank_point(const DevPlan &P, const UnrankTabs &U, unsigned long long r, int *K, int *Lv, int *J,
                            int &bout) {
    const int d = P.d, L = P.L, W = d + 1;
    if (r >= U.shard_points) return -1;
    auto counted = [&](int b) { return U.merge || P.coef[b] != 0.0; };
    bout = 0;
    if (U.include_root && counted(0)) {
        if (r == 0) return 0;
        r -= 1;
    }
    // depth-1 prefix: largest i with D1[i] <= r (binary search over the shard's r1 range)
    long long a = 0, e = U.n1;
    while (e - a > 1) {
        const long long m = (a + e) >> 1;
        if (U.D1[m] <= r) a = m;
        else e = m;
    }
    r -= U.D1[a];
    const long long r1 = U.lo + a;
    const int k1 = (int)(r1 / P.M0);
    int rem = (int)(r1 - (long long)k1 * P.M0), l1 = 2;
    while (rem >= P.nl[l1]) {
        rem -= P.nl[l1];
        ++l1;
    }
    K[0] = k1;
    Lv[0] = l1;
    J[0] = rem;
    int depth = 1, b = l1 - 1, kl = k1;
    for (;;) {
        if (counted(b)) {
            if (r == 0) break;
            r -= 1;
        }
        // coordinate kp: largest kp in [kl+1, d) with SG[b][kl+1] - SG[b][kp] <= r
        const unsigned long long base = U.SG[(size_t)b * W + kl + 1];
        int lo = kl + 1, hi = d;   // invariant: cum(lo) <= r, answer in [lo, hi)
        while (hi - lo > 1) {
            const int m = (lo + hi) >> 1;
            if (base - U.SG[(size_t)b * W + m] <= r) lo = m;
            else hi = m;
        }
        r -= base - U.SG[(size_t)b * W + lo];
        int lp = 2;
        for (; lp <= L + 1 - b; ++lp) {
            const unsigned long long s = U.Sub[(size_t)(b + lp - 1) * W + lo + 1];
            const unsigned long long blk = (unsigned long long)P.nl[lp] * s;
            if (r < blk) {
                J[depth] = (int)(r / s);
                r %= s;
                break;
            }
            r -= blk;
        }
        if (lp > L + 1 - b) return -1;   // inconsistent tables (cannot happen)
        K[depth] = lo;
        Lv[depth] = lp;
        ++depth;
        b += lp - 1;
        kl = lo;
    }
    bout = b;
    return depth;
}

// One thread per index: unrank, then the point's term c(t, b) * Re(B * prod_m F[l_m][k_m][j_m]) in
// (complex) double-double, straight from the factor table — an evaluation independent of the
// prefix tree's partial products and accumulators.
__global__ void __launch_bounds__(128) k_eval_points(const DevPlan P, const UnrankTabs U,
                                                     const unsigned long long *idx, long long n, int *pts,
                                                     double *out) {
    const long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    int K[SG_MAX_L + 1], Lv[SG_MAX_L + 1], J[SG_MAX_L + 1], b = 0;
    const int t = unrank_point(P, U, idx[i], K, Lv, J, b);
    const int stride = 1 + 3 * P.L;
    int *rec = pts + i * stride;
    rec[0] = t;
    for (int m = 0; m < P.L; ++m) {
        rec[1 + 3 * m] = m < t ? K[m] : -1;
        rec[2 + 3 * m] = m < t ? Lv[m] : -1;
        rec[3 + 3 * m] = m < t ? J[m] : -1;
    }
    if (t < 0) {
        out[2 * i] = nan("");
        out[2 * i + 1] = nan("");
        return;
    }
    cdd v = {dd{P.base[0], P.base[1]}, dd{P.base[2], P.base[3]}};
    for (int m = 0; m < t; ++m) {
        const int e = P.tab_off[Lv[m]] + K[m] * P.nl[Lv[m]] + J[m];
        const double2 fr = P.Fre[e];
        const double2 fi = P.Fim ? P.Fim[e] : make_double2(0.0, 0.0);
        v = cdd_mul(v, cdd{dd{fr.x, fr.y}, dd{fi.x, fi.y}});
    }
    const double2 c = P.coefm[t * (P.L + 1) + b];
    const dd term = dd_mul(v.re, dd{c.x, c.y});
    out[2 * i] = term.hi;
    out[2 * i + 1] = term.lo;
}

// SG_METHOD_PLAIN: every point evaluated independently (the paper's plain SG baseline, no dimension
// iteration): thread g handles the flat indices g, g + G, g + 2G, ... of the shard (fixed order),
// unranks each one and forms its term from its t factors; dd accumulation, fixed CTA reduction.
__global__ void __launch_bounds__(256) k_plain(const DevPlan P, const UnrankTabs U, double2 *partials) {
    const unsigned long long G = (unsigned long long)gridDim.x * blockDim.x;
    const unsigned long long g0 = (unsigned long long)blockIdx.x * blockDim.x + threadIdx.x;
    double ah = 0.0, al = 0.0;
    int K[SG_MAX_L + 1], Lv[SG_MAX_L + 1], J[SG_MAX_L + 1];
    const cdd B = {dd{P.base[0], P.base[1]}, dd{P.base[2], P.base[3]}};
    for (unsigned long long i = g0; i < U.shard_points; i += G) {
        int b = 0;
        const int t = unrank_point(P, U, i, K, Lv, J, b);
        if (t < 0) continue;
        cdd v = B;
        for (int m = 0; m < t; ++m) {
            const int e = P.tab_off[Lv[m]] + K[m] * P.nl[Lv[m]] + J[m];
            const double2 fr = P.Fre[e];
            const double2 fi = P.Fim ? P.Fim[e] : make_double2(0.0, 0.0);
            v = cdd_mul_fast(v, cdd{dd{fr.x, fr.y}, dd{fi.x, fi.y}});
        }
        const double2 c = P.coefm[t * (P.L + 1) + b];
        double p, e;
        dd_mul_pe(v.re, dd{c.x, c.y}, p, e);
        acc_add(ah, al, p, e);
    }
    const dd s = block_reduce_dd<8>(dd_norm(ah, al));
    if (threadIdx.x == 0) SG_PART(partials, blockIdx.x) = make_double2(s.hi, s.lo);
}
