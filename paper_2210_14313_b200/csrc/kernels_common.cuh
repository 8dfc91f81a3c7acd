// kernels_common.cuh — device-side plan/argument structs, warp/CTA dd reductions (K4) and the dd helpers shared by every kernel
// (included once, by sg_kernels.cu, after the shared definitions it uses)
#pragma once

#define WPB 8                 // warps per CTA in the pass kernels
#define PASS_THREADS (WPB * 32)
#define META_KMASK ((1u << SG_META_KBITS) - 1u)

// task descriptor words (plan.cpp pack32): two int32 fields, the high one possibly negative
__device__ __forceinline__ int task_hi32(long long v) { return (int)(int32_t)(uint32_t)((unsigned long long)v >> 32); }
__device__ __forceinline__ int task_lo32(long long v) { return (int)(int32_t)(uint32_t)((unsigned long long)v & 0xffffffffull); }

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
    double wabs[SG_MAX_L + 3];   // sum_j |w_j^l| (+ |lo|) per level: k_head's analytic suffix bounds
};

// ---------------------------------------------------------------------------------------------
// Checked build (-DSG_CHECKS, tools/checked_run.py; compute-sanitizer is closed on this GPU pool):
// every frontier read / write is bounds-checked against its buffer's capacity, every partial slot
// write is counted (each slot must be written exactly once per step: a task claimed twice or never
// shows up there), and the first violation is recorded.  The production build compiles the same
// accessors to plain indexing (no fields, no code).
// ---------------------------------------------------------------------------------------------
#ifdef SG_CHECKS
#define SG_CHK_FIELDS long long chk_src_cap, chk_dst_cap;
struct ChkState {
    unsigned long long viol;
    long long first[4];   // code, index, bound, source line of the first violation
    unsigned *writes;     // write count per partial slot
    long long nslots;
    const double2 *part_base;
};
__device__ ChkState g_chk;
__device__ __noinline__ void chk_fail(int code, long long idx, long long bound, int line) {
    if (atomicAdd(&g_chk.viol, 1ull) == 0) {
        g_chk.first[0] = code;
        g_chk.first[1] = idx;
        g_chk.first[2] = bound;
        g_chk.first[3] = line;
    }
}
template <class T>
__device__ __forceinline__ T *chk_at(T *p, long long i, long long cap, int code, int line) {
    if (i < 0 || i >= cap) chk_fail(code, i, cap, line);
    return p;
}
__device__ __forceinline__ double2 *chk_part(double2 *p, int line) {
    const long long sl = (long long)(p - g_chk.part_base);
    if (!g_chk.writes || sl < 0 || sl >= g_chk.nslots) chk_fail(3, sl, g_chk.nslots, line);
    else atomicAdd(g_chk.writes + sl, 1u);
    return p;
}
#define SG_SRC(A, f, i) (*chk_at(&(A).f[i], (long long)(i), (A).chk_src_cap, 1, __LINE__))
#define SG_DST(A, f, i) (*chk_at(&(A).f[i], (long long)(i), (A).chk_dst_cap, 2, __LINE__))
#define SG_PART(base, i) (*chk_part(&(base)[i], __LINE__))
#define SG_CHK(i, cap, code) ((void)chk_at((const char *)nullptr, (long long)(i), (long long)(cap), code, __LINE__))
#else
#define SG_CHK_FIELDS
#define SG_SRC(A, f, i) ((A).f[i])
#define SG_DST(A, f, i) ((A).f[i])
#define SG_PART(base, i) ((base)[i])
#define SG_CHK(i, cap, code) ((void)0)
#endif

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
    int stage_lmax;                // k_pass: factor levels 2 .. stage_lmax staged in shared memory
    int stage_entries;             // their table entries (d * sum nl)
    SG_CHK_FIELDS
};

struct RootArgs {
    long long lo, hi;
    const long long *off1, *JS;
    double2 *dst_re, *dst_im;
    uint32_t *dst_meta;
    double2 *partials;
    SG_CHK_FIELDS
};

// Status words: status[0] is the live NonFiniteIntegrand flag of the running step (atomicOr by any
// kernel), status[1] the flag of the last completed sg_integrate (read by k_finalize and
// sg_status_word).  The step's final kernel publishes status[0] to status[1] and clears status[0],
// so every sg_integrate starts with a clear flag without a memset node.
__device__ __forceinline__ void step_close_status(const DevPlan &P, int st) {
    P.status[1] = st ? 1 : 0;
    P.status[0] = 0;
}

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
// leaf arithmetic helpers
// ---------------------------------------------------------------------------------------------
// Biased grid accumulator start value for a lane whose terms sum to at most `bound` in magnitude:
// sigma = 1.5 * 2^e with 2^e > 2 * bound, i.e. 3 * (the power of two <= 2 * bound), taken from the
// exponent bits (at least 3 * the smallest normal, so a zero bound still gives a positive sigma).
// Measured on config 5: the fused leaf kernel 12.29 -> 12.15 ms against frexp / ldexp.
__device__ __forceinline__ double grid_sigma(double bound) {
    const int hi = max(__double2hiint(2.0 * bound) & 0x7ff00000, 0x00100000);
    return 3.0 * __hiloint2double(hi, 0);
}
// The same sigma (1.5 for a zero bound) by frexp / ldexp.
__device__ __forceinline__ double grid_sigma_frexp(double bound) {
    int ex = 0;
    frexp(2.0 * bound, &ex);
    return bound > 0.0 ? ldexp(1.5, ex) : 1.5;
}

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

