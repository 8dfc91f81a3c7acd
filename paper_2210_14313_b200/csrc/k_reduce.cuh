// k_reduce.cuh — K4/K5: fixed-order reductions of the task partials and the cross-rank finalize
// (included once, by sg_kernels.cu, after the shared definitions it uses)
#pragma once

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

__global__ void k_finalize(const double *gathered, int world, const int *status, double *result) {
    if (threadIdx.x != 0 || blockIdx.x != 0) return;
    dd s = {0.0, 0.0};
    for (int r = 0; r < world; ++r) s = dd_add(s, dd{gathered[2 * r], gathered[2 * r + 1]});
    if (*status || !isfinite(s.hi)) s = dd{nan(""), nan("")};
    result[0] = s.hi;
    result[1] = s.lo;
}

