// k_head.cuh — the head of a step in ONE cooperative launch: K0 (factor table and base), then, after a
// grid-wide barrier, the root pass and the suffix bounds of |F| (independent of each other).
// (included once, by sg_kernels.cu, after k_factor.cuh and k_tree.cuh)
#pragma once
#include <cooperative_groups.h>

// Replaces k_factor_base + k_suffix_abs + k_root (three graph nodes, ~30 us of fixed work per step
// on configs 4-5 measured in-graph) when every block of the grid is co-resident (cooperative launch;
// the host checks the occupancy) and d <= HEAD_SUF_MAXCH * K0_THREADS (suffix rows per thread held in
// registers).  Block b: phase A = factor entries [256 b, 256 b + 256) (b < nfb) or the base (b == nfb);
// phase B = the root points r1 = lo + 256 b + t (b < root_blocks, partial per block as in k_root),
// and for b < L the suffix bounds SA of level 2 + b.  Same arithmetic and summation orders as the
// three kernels it replaces: bitwise the same results.
#define HEAD_SUF_MAXCH 8

__device__ __forceinline__ void head_suffix_level(const DevPlan &P, int l, double *suf) {
    const int d = P.d, n = P.nl[l];
    const double2 *Fr = P.Fre + P.tab_off[l];
    const double2 *Fi = P.kind == SG_F_OSCILLATORY ? P.Fim + P.tab_off[l] : nullptr;
    const int chunk = (d + K0_THREADS - 1) / K0_THREADS;   // <= HEAD_SUF_MAXCH (host-checked)
    const int k0 = min(d, (int)threadIdx.x * chunk), k1 = min(d, k0 + chunk);
    // row sums of this thread's rows, every load issued before any is consumed (F was written by other
    // blocks before the grid barrier: L2 loads, not the non-coherent path)
    double rs[HEAD_SUF_MAXCH];
#pragma unroll
    for (int c = 0; c < HEAD_SUF_MAXCH; ++c) rs[c] = 0.0;
    for (int j = 0; j < n; ++j) {
#pragma unroll
        for (int c = 0; c < HEAD_SUF_MAXCH; ++c) {
            const int k = k0 + c;
            if (k < k1) {
                rs[c] += fabs(__ldcg(Fr + (long long)k * n + j).x);
                if (Fi) rs[c] += fabs(__ldcg(Fi + (long long)k * n + j).x);
            }
        }
    }
    double cs = 0.0;
#pragma unroll
    for (int c = 0; c < HEAD_SUF_MAXCH; ++c) cs += rs[c];
    suf[threadIdx.x] = cs;
    if (threadIdx.x == 0) suf[K0_THREADS] = 0.0;
    __syncthreads();
    for (int off = 1; off < K0_THREADS; off <<= 1) {   // suf[i] = sum of chunks i.. end
        const double t = (threadIdx.x + off < K0_THREADS) ? suf[threadIdx.x + off] : 0.0;
        __syncthreads();
        suf[threadIdx.x] += t;
        __syncthreads();
    }
    double sacc = suf[threadIdx.x + 1];
    if (threadIdx.x == 0) P.SA[(long long)l * (d + 1) + d] = 0.0;
#pragma unroll
    for (int c = HEAD_SUF_MAXCH - 1; c >= 0; --c) {
        const int k = k0 + c;
        if (k < k1) {
            sacc += rs[c];
            P.SA[(long long)l * (d + 1) + k] = sacc;
        }
    }
}

template <bool CPLX>
__global__ void __launch_bounds__(K0_THREADS) k_head(const DevPlan P, const RootArgs R, int nfb, int root_blocks) {
    const int b = blockIdx.x;
    // phase A: K0
    if (b == nfb) base_body(P);
    else if (b < nfb) factor_entry(P, b * K0_THREADS + threadIdx.x);
    cooperative_groups::this_grid().sync();
    // phase B: root pass (needs F and B) and suffix bounds (need F)
    if (b < root_blocks) {
        const long long r1 = R.lo + (long long)b * K0_THREADS + threadIdx.x;
        dd s = block_reduce_dd<K0_THREADS / 32>(root_node<CPLX>(P, R, r1));
        if (threadIdx.x == 0) R.partials[b] = make_double2(s.hi, s.lo);
    }
    if (b < P.L) {
        __shared__ double suf[K0_THREADS + 1];
        __syncthreads();
        head_suffix_level(P, 2 + b, suf);
    }
}
