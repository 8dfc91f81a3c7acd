// k_reduce.cuh — K4/K5: fixed-order reductions of the task partials and the cross-rank finalize
// (included once, by sg_kernels.cu, after the shared definitions it uses)
#pragma once

// One-block fixed-order reduction of per-block partials (+ the root point) -> out[0..1] (plain path).
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
        const int st = *P.status;
        if (st) s = dd{nan(""), nan("")};
        out[0] = s.hi;
        out[1] = s.lo;
        step_close_status(P, st);
    }
}

// Tree-path reduction in ONE launch: block b sums partials [b*RED_CHUNK2, (b+1)*RED_CHUNK2) (each
// thread its RED_PER_THREAD elements, loads issued together, summed in index order), writes l1[b];
// the last block to finish (atomic ticket after a fence) sums l1[0..nblk) in a fixed order, adds the
// root point and writes out[0..1], then re-arms the ticket.  Which block is last does not change any
// summation order, so the result is bitwise reproducible.
#define RED_THREADS 256
#define RED_PER_THREAD 8
#define RED_CHUNK2 (RED_THREADS * RED_PER_THREAD)
// SF = DevPlan::sform (0 factor form, 1 / 2 s-forms): the root point's value; one instantiation each
// keeps the s-forms' per-point outer functions out of the factor-form launch (instruction fetch)
template <int SF>
__global__ void __launch_bounds__(RED_THREADS)
k_reduce_fused(const DevPlan P, const double2 *partials, long long n, int include_root, double *out,
               double2 *l1, unsigned long long *ticket, unsigned long long *task_counters) {
    const long long b0 = (long long)blockIdx.x * RED_CHUNK2 + (long long)threadIdx.x * RED_PER_THREAD;
    double2 v[RED_PER_THREAD];
#pragma unroll
    for (int i = 0; i < RED_PER_THREAD; ++i)
        v[i] = b0 + i < n ? __ldcg(partials + b0 + i) : make_double2(0.0, 0.0);
    dd s = {0.0, 0.0};
#pragma unroll
    for (int i = 0; i < RED_PER_THREAD; ++i) s = dd_add(s, dd{v[i].x, v[i].y});
    s = block_reduce_dd<RED_THREADS / 32>(s);
    __shared__ int last;
    if (threadIdx.x == 0) {
        l1[blockIdx.x] = make_double2(s.hi, s.lo);
        __threadfence();
        last = atomicAdd(ticket, 1ULL) == (unsigned long long)gridDim.x - 1;
    }
    __syncthreads();
    if (!last) return;
    __threadfence();
    dd t = {0.0, 0.0};
    for (unsigned i = threadIdx.x; i < gridDim.x; i += RED_THREADS) {
        const double2 x = __ldcg(l1 + i);
        t = dd_add(t, dd{x.x, x.y});
    }
    __syncthreads();   // the block_reduce scratch is reused
    t = block_reduce_dd<RED_THREADS / 32>(t);
    if (threadIdx.x == 0) {
        if (include_root && P.coefm[0].x != 0.0) {
            const dd root = SF == 2   ? sform_g_dd(P.kind, P.d, dd{P.base[0], P.base[1]})
                            : SF == 1 ? dd{sform_g(P.kind, P.d, P.base[0]), 0.0}
                                      : dd{P.base[0], P.base[1]};
            t = dd_add(t, coef_mul(P, root, 0, 0));
        }
        const int st = *P.status;
        if (st) t = dd{nan(""), nan("")};
        out[0] = t.hi;
        out[1] = t.lo;
        *ticket = 0;
        // re-arm the persistent leaf kernels' task counters for the next step (all of this step's
        // passes finished before this launch)
        task_counters[0] = 0;
        task_counters[2] = 0;
        task_counters[4] = 0;
        step_close_status(P, st);
    }
}

// status = the plan's status words; status[1] holds the flag of the last completed sg_integrate
__global__ void k_finalize(const double *gathered, int world, const int *status, double *result) {
    if (threadIdx.x != 0 || blockIdx.x != 0) return;
    dd s = {0.0, 0.0};
    for (int r = 0; r < world; ++r) s = dd_add(s, dd{gathered[2 * r], gathered[2 * r + 1]});
    if (status[1] || !isfinite(s.hi)) s = dd{nan(""), nan("")};
    result[0] = s.hi;
    result[1] = s.lo;
}

