// sg_kernels.cu — the single CUDA translation unit of the B200 Smolyak hot path: the kernels (in the
// headers below, one per stage) and the C ABI of include/sg_b200.h (plan object, launches).
//
//  kernels_common.cuh  device plan/argument structs, fixed-order dd warp/CTA reductions (K4)
//  k_factor.cuh        K0: factor table F = w * E_k(x) and base B in double-double,
//                      suffix bounds of |F| for the leaf kernels' grid accumulators
//  k_tree.cuh          K2+K3: level-synchronous prefix-tree passes (Eqs 3.8-3.11,
//                      the multilevel dimension iteration): root pass, frontier writer k_pass,
//                      leaf kernels k_leaf (generic), k_leaf1 (single level), k_leaf2 / _pairs /
//                      _sym3 (fused last two levels, the hot loop; k_leaf2_sym3<SRC> also runs
//                      pass L-2 as source tasks)
//  k_sform.cuh         s-form passes (partial sums of the argument, outer function per point)
//  k_unrank.cuh        device unranker (sg_eval_points) and the plain per-point SG ablation
//  k_reduce.cuh        K4/K5: task partials -> fixed-order dd sum; cross-rank finalize
//  k_collapse.cuh      separable collapse (SG_METHOD_COLLAPSE)
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

#include "kernels_common.cuh"
#include "k_factor.cuh"
#include "k_tree.cuh"
#include "k_sform.cuh"
#include "k_reduce.cuh"
#include "k_collapse.cuh"
#include "k_unrank.cuh"

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
    void *d_unrank = nullptr;  // sg_eval_points: device Sub / SG / D1 tables (built on first use)
    UnrankTabs utabs = {};
    bool plain = false;        // SG_METHOD_PLAIN: every point unranked and evaluated on its own
    int plain_blocks = 0;
    bool collapse = false;     // SG_METHOD_COLLAPSE: O(d L^2) per-coordinate polynomial product
    int collapse_blocks = 0;   // CTAs of k_collapse_part (one partial polynomial each)
    bool collapse_emit = true; // rank 0 emits the value; other ranks contribute 0
    // plan-owned device memory
    void *dev_block = nullptr;
    size_t dev_bytes = 0;
    long long *d_tabs = nullptr;
    std::vector<size_t> tab_offT, tab_NT, tab_CT, tab_TB;   // element offsets into d_tabs per depth
    size_t tab_JS = 0, tab_off1 = 0, tab_TK = 0, tab_TKS = 0;
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
    int leaf2_threads = PASS_THREADS;   // CTA size of the persistent leaf launch
    int leaf2_l3s = 0;                  // level-3 row symmetry for the source tasks (0 / 1 / 2)
    bool head = false;                  // K0 + base + root + suffix bounds as one k_head launch
    int prof_mode = 0;                  // sg_profile_enable: 1 every launch, 2 the dominant pass only
    int prof_dom = -1;                  // the dominant pass (most points)
    int world = 1;                      // shard count of the plan's partition (options)
    size_t pass_smem_cap = 0;           // k_pass: bytes of factor levels staged in shared memory
                                        // (SG_B200_PASS_SMEM: A/B runs)
    int prefetch_min = 16;              // fused kernel prefetches the next task with >= this many
                                        // tasks per resident warp (SG_B200_PREFETCH_MIN: A/B runs)
    std::vector<cudaEvent_t> ev;
    std::vector<std::pair<int, int>> prof_pairs;   // per launch of the last sg_integrate: (start, end) event
    // fused plans: pass nfront-1 runs on a plan-owned side stream, concurrently with the fused pass
    cudaStream_t side = nullptr;
    // split frontier passes: the runs of the stored children (k_front), per pass t (plan-owned)
    FrontChunk *d_runs = nullptr;
    std::vector<long long> runs_off, runs_n;   // per pass t: offset into d_runs (chunks), count
    int front_grid = 0;                        // k_front CTAs (persistent)
    std::vector<FrontChunk> front_chunks;      // host copy (built with the partial layout)
    bool split_serial = false;                 // leaf-only kernel after k_front on the same stream
    bool fork1 = false;                        // passes L-2 || L-1 concurrent at world 1 too (see sg_integrate)
    int resident_ctas = 0;                     // fused launch: SMs x CTAs per SM (setup_leaf1)
    cudaEvent_t ev_fork = nullptr, ev_join = nullptr;
    // workspace
    char *ws = nullptr;
    size_t ws_bytes = 0;
    size_t ws_front_off[2] = {0, 0}, ws_part_off = 0, ws_red_off = 0, ws_need = 0;
};

static size_t align_up(size_t x, size_t a) { return (x + a - 1) / a * a; }

// Partial slots: the root's, then per pass t its pass_blocks[t] (twice for a split frontier pass).
#define FRONT_GRID 148   // k_front CTAs (persistent, one per SM: A/B r02z serial 148 -> 1.45 ms, 592 -> 1.65 ms)
// split pass t: slots [0, pass_split[t] - 1) for k_front's chunks, then pass_blocks[t] for k_leaf
static void layout_partials(HostPlan &hp) {
    int64_t poff = hp.root_blocks;
    for (int u = 1; u <= hp.nfront; ++u) {
        hp.pass_partial_off[u] = poff;
        const int64_t fs = u < (int)hp.pass_front_slots.size() ? hp.pass_front_slots[u] : 0;
        poff += hp.pass_blocks[u] + fs;
    }
    hp.total_partials = poff;
}

// Source chunks of pass t for k_front: every segment (b <= L-2: it has stored children) of frontier t
// cut into chunks of FRONT_THREADS * FRONT_SPT consecutive sources.
static void build_front_chunks(const HostPlan &hp, int t, std::vector<FrontChunk> &ch) {
    const int d = hp.d, L = hp.L;
    for (int b = 0; b <= L - 2; ++b)
        for (int k = 0; k <= d - 3; ++k) {   // a stored child needs a row k' in (k, d-2]
            const int64_t N = hp.N[t][(size_t)b * d + k];
            for (int64_t i0 = 0; i0 < N; i0 += FRONT_THREADS * FRONT_SPT)
                ch.push_back(FrontChunk{hp.off[t][(size_t)b * d + k] + i0, (int)i0,
                                        (int)std::min<int64_t>(FRONT_THREADS * FRONT_SPT, N - i0), b, k,
                                        hp.C[t][(size_t)b * d + k], N});
        }
}
static int setup_leaf1(sg_plan_s *p);
static int build_unrank_tables(sg_plan_s *p);

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
    if (o.method != SG_METHOD_TREE && o.method != SG_METHOD_COLLAPSE && o.method != SG_METHOD_PLAIN)
        return SG_EINVAL;
    if (o.method == SG_METHOD_PLAIN && o.arith != SG_ARITH_FACTOR_DD) return SG_EUNSUPPORTED;
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
        if (o.arith != SG_ARITH_FACTOR_DD || o.method == SG_METHOD_PLAIN) mode = 0;
        p->plain = (o.method == SG_METHOD_PLAIN);
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
    p->world = (o.range_hi > o.range_lo && o.range_lo >= 0) ? 2 : o.world;   // explicit range: a shard
    for (int t = 1; t <= hp.nfront; ++t)
        if (p->prof_dom < 0 || hp.pass_terms[t] > hp.pass_terms[p->prof_dom]) p->prof_dom = t;
    p->sform = (o.arith == SG_ARITH_SFORM_FP64 || o.arith == SG_ARITH_SFORM_DD);
    p->sform_dd = (o.arith == SG_ARITH_SFORM_DD);
    p->two = p->cplx || p->sform;
    {
        // specialised single-level / fused leaf kernels: factor form only; SG_B200_GENERIC_LEAF=1
        // forces the generic k_leaf (tests)
        const char *g = getenv("SG_B200_GENERIC_LEAF");
        p->leaf1 = !p->sform && !(g && g[0] == '1');
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
    if (hp.leaf2_srctasks) p->tab_TKS = push(hp.T2S);
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
    for (int l = 2; l <= L + 1; ++l) {   // sum_j |w_j^l| of the level's table entries (k_head's SA bound)
        double a = 0.0;
        for (int j = 0; j < hp.nl[l]; ++j) a += fabs(hp.Whi[hp.entry_off[l] + j]) + fabs(hp.Wlo[hp.entry_off[l] + j]);
        dp.wabs[l] = a;
    }
    dp.M0 = hp.M0;
    dp.symmask = 0;
    for (int l = 2; l <= L + 1; ++l) {
        const int n = hp.nl[l], e0 = hp.entry_off[l];
        bool sym = n >= 2 && (n % 2 == 0 || hp.X[e0 + n / 2] == 0.5);
        for (int j = 0; sym && j < n / 2; ++j) {
            const int m = e0 + n - 1 - j;
            sym = (1.0 - hp.X[m] == hp.X[e0 + j]) && hp.Whi[m] == hp.Whi[e0 + j] && hp.Wlo[m] == hp.Wlo[e0 + j];
        }
#ifndef LEAF_NO_SYMROWS
        if (sym) dp.symmask |= 1 << l;
#endif
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
    ok &= cudaMemset(p->d_counter, 0, sizeof(unsigned long long) * 8) == cudaSuccess;   // tickets
    ok &= cudaMemcpy((void *)dp.coefm, cm.data(), sizeof(double2) * cm.size(), cudaMemcpyHostToDevice) == cudaSuccess;
    if (!ok) {
        cudaGetLastError();
        cudaFree(p->dev_block);
        delete p;
        return SG_ECUDA;
    }
    if (const char *e = getenv("SG_B200_PREFETCH_MIN"); e && e[0]) p->prefetch_min = atoi(e);
    {
        // Split frontier passes (factor form): a pass that stores more than FRONT_SPLIT_MIN_BYTES of
        // frontier records runs as a write-only k_pass (the stored children, their terms from the
        // stored products) and, concurrently on the side stream, a leaf-only k_leaf (the other
        // children).  SG_B200_FRONT_SPLIT=0/1 forces it off/on (A/B, tests).
        const char *e = getenv("SG_B200_FRONT_SPLIT"), *nf = getenv("SG_B200_NOFORK");
        const int force = (nf && nf[0] == '1') ? 0 : (e && e[0]) ? atoi(e) : -1;   // no side stream: no split
        hp.pass_split.assign(hp.nfront + 1, 0);
        const size_t rec = (p->cplx ? 32 : 16) + 4;
        for (int t = 1; t < hp.nfront; ++t) {
            const bool writes = !(hp.fuse && t + 1 == hp.nfront);
            const bool big = (double)hp.pass_written[t] * rec >= FRONT_SPLIT_MIN_BYTES;
            // k_front indexes a source inside its segment with an int (FrontChunk::i0)
            bool fits = true;
            for (size_t q = 0; q < hp.N[t].size(); ++q) fits = fits && hp.N[t][q] < INT_MAX;
            if (!fits) continue;
            hp.pass_split[t] = (!p->sform && writes && (force == 1 || (force != 0 && big))) ? 1 : 0;
        }
        // k_front chunks of the split passes (heavy-first: work ~ sources x rows x stored nodes)
        hp.pass_front_slots.assign(hp.nfront + 1, 0);
        p->runs_off.assign(hp.nfront + 1, 0);
        p->runs_n.assign(hp.nfront + 1, 0);
        p->front_chunks.clear();
        for (int t = 1; t < hp.nfront; ++t) {
            if (!hp.pass_split[t]) continue;
            std::vector<FrontChunk> ch;
            build_front_chunks(hp, t, ch);
            auto work = [&](const FrontChunk &c) {
                int64_t nodes = 0;
                for (int lp = 2; lp <= hp.L - c.b; ++lp) nodes += hp.nl[lp];
                return (int64_t)c.cnt * (hp.d - 2 - c.k) * nodes;
            };
            std::stable_sort(ch.begin(), ch.end(), [&](const FrontChunk &a, const FrontChunk &b2) {
                return work(a) > work(b2);
            });
            p->runs_off[t] = (long long)p->front_chunks.size();
            p->runs_n[t] = (long long)ch.size();
            hp.pass_front_slots[t] = (int64_t)ch.size();
            p->front_chunks.insert(p->front_chunks.end(), ch.begin(), ch.end());
        }
        layout_partials(hp);
    }
    if (const char *e = getenv("SG_B200_PASS_SMEM"); e && e[0]) p->pass_smem_cap = (size_t)atoll(e);
    if (p->pass_smem_cap > 48 * 1024) {
        if (cudaFuncSetAttribute(k_pass<true, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024) != cudaSuccess ||
            cudaFuncSetAttribute(k_pass<false, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024) != cudaSuccess) {
            cudaGetLastError();
            p->pass_smem_cap = 48 * 1024;
        }
        p->pass_smem_cap = std::min<size_t>(p->pass_smem_cap, 200 * 1024);
    }
    rc = (p->collapse || p->plain) ? SG_OK : setup_leaf1(p);
    if (rc) {
        cudaGetLastError();
        cudaFree(p->dev_block);
        delete p;
        return rc;
    }
    if (p->plain) {
        // ---- plain per-point method: unrank tables (plan-owned), one dd partial per CTA ----
        rc = build_unrank_tables(p);
        if (rc) {
            cudaFree(p->dev_block);
            delete p;
            return rc;
        }
        int dev = 0, sms = 148;
        cudaGetDevice(&dev);
        cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
        p->plain_blocks = sms * 8;
        p->ws_part_off = 0;
        p->ws_red_off = align_up(sizeof(double2) * (size_t)p->plain_blocks, 256);
        p->ws_need = p->ws_red_off + 256;
        *out = p;
        return SG_OK;
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
    ws = align_up(ws + sizeof(double2) * (size_t)((hp.total_partials + RED_CHUNK2 - 1) / RED_CHUNK2 + 1), 256);
    p->ws_need = ws;
    {
        // one head launch for the factor form at d <= HEAD_MAX_D; SG_B200_NOHEAD=1 keeps the three
        // launches (A/B, tests)
        const char *nh = getenv("SG_B200_NOHEAD");
        p->head = !p->sform && hp.d <= HEAD_MAX_D && !(nh && nh[0] == '1');
    }
    bool any_split = false;
    for (size_t t = 0; t < hp.pass_split.size(); ++t) any_split = any_split || hp.pass_split[t];
    if (any_split) {
        const std::vector<FrontChunk> &runs = p->front_chunks;
        p->front_grid = FRONT_GRID;
        if (const char *e = getenv("SG_B200_FRONT_GRID"); e && e[0]) p->front_grid = std::max(1, atoi(e));   // A/B
        p->split_serial = getenv("SG_B200_SPLIT_SERIAL") && getenv("SG_B200_SPLIT_SERIAL")[0] == '1';
        if (cudaMalloc(&p->d_runs, sizeof(FrontChunk) * std::max<size_t>(runs.size(), 1)) != cudaSuccess ||
            cudaMemcpy(p->d_runs, runs.data(), sizeof(FrontChunk) * runs.size(), cudaMemcpyHostToDevice) != cudaSuccess) {
            cudaGetLastError();
            sg_destroy(p);
            return SG_ENOMEM;
        }
    }
    // world 1: fork only when the fused launch leaves SMs free (its grid is below the resident CTAs);
    // a full persistent grid would have to wait for the concurrent pass's CTAs to drain on every SM
    // they took (config 3: 0.085 -> 0.087 ms forked; configs 1-2: 0.038 -> 0.036, 0.109 -> 0.097 ms)
    p->fork1 = p->leaf2 && p->leaf1_grid < p->resident_ctas;
    if (const char *e = getenv("SG_B200_FORK1"); e && e[0]) p->fork1 = e[0] == '1';   // A/B
    if ((any_split || (p->leaf2 && hp.nfront >= 2 && (p->world > 1 || p->fork1))) &&
        !(getenv("SG_B200_NOFORK") && getenv("SG_B200_NOFORK")[0] == '1')) {
        // side stream + fork/join events for the concurrent passes nfront-1 and nfront (sg_integrate)
        // highest priority: the shorter pass's blocks are scheduled first, the persistent fused kernel
        // fills the rest of the GPU and takes over the SMs the short pass frees (graph kernel nodes
        // keep the capturing stream's priority)
        int prio_lo = 0, prio_hi = 0;
        cudaDeviceGetStreamPriorityRange(&prio_lo, &prio_hi);
        if (cudaStreamCreateWithPriority(&p->side, cudaStreamNonBlocking, prio_hi) != cudaSuccess ||
            cudaEventCreateWithFlags(&p->ev_fork, cudaEventDisableTiming) != cudaSuccess ||
            cudaEventCreateWithFlags(&p->ev_join, cudaEventDisableTiming) != cudaSuccess) {
            cudaGetLastError();
            sg_destroy(p);
            return SG_ECUDA;
        }
    }
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
// Real kinds with few parents per shard: lane groups (k_leaf2 G = 2, 4, 8; plan.cpp leaf2_groups)
template <bool SMEM, int G>
static const void *leaf2_fn_groups(int nj, bool center, bool cz) {
    if (nj == 3 && center)
        return cz ? (const void *)k_leaf2<false, 3, SMEM, 1, false, true, G> : (const void *)k_leaf2<false, 3, SMEM, 1, false, false, G>;
    if (nj == 3) return (const void *)k_leaf2<false, 3, SMEM, -1, false, false, G>;
    return (const void *)k_leaf2<false, 2, SMEM, -1, false, false, G>;
}

template <bool CPLX, bool SMEM>
static const void *leaf2_fn(int nj, bool center, bool sym, bool cz, int groups = 1) {
    if (!CPLX && groups == 2) return leaf2_fn_groups<SMEM, 2>(nj, center, cz);
    if (!CPLX && groups == 4) return leaf2_fn_groups<SMEM, 4>(nj, center, cz);
    if (!CPLX && groups == 8) return leaf2_fn_groups<SMEM, 8>(nj, center, cz);
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
static const void *leaf2_kernel(int nj, bool smem, bool center, bool sym, bool cz, int ppl = 1, int groups = 1) {
    if (CPLX && sym && center && nj == 3 && ppl >= 2) {
#define SYM3(P_) (smem ? (cz ? (const void *)k_leaf2_sym3<P_, true, true, false> : (const void *)k_leaf2_sym3<P_, true, false, false>) \
                       : (cz ? (const void *)k_leaf2_sym3<P_, false, true, false> : (const void *)k_leaf2_sym3<P_, false, false, false>))
        if (ppl == 2) return SYM3(2);
        if (ppl == 3) return SYM3(3);
#undef SYM3
    }
    if (CPLX && sym && nj == 2 && ppl == 2)
        return smem ? (const void *)k_leaf2_pairs<2, true> : (const void *)k_leaf2_pairs<2, false>;
    if (CPLX && sym && nj == 2 && ppl == 3)
        return smem ? (const void *)k_leaf2_pairs<3, true> : (const void *)k_leaf2_pairs<3, false>;
    if (CPLX && sym && nj == 2 && ppl == 4)
        return smem ? (const void *)k_leaf2_pairs<4, true> : (const void *)k_leaf2_pairs<4, false>;
    return smem ? leaf2_fn<CPLX, true>(nj, center, sym, cz, groups) : leaf2_fn<CPLX, false>(nj, center, sym, cz, groups);
}

// The source-task kernel of pass L-2 (plan.cpp builds source tasks only for k_leaf2_sym3 plans, with
// LEAF2_PPL3 parents per lane); l3s = symmetry of the level-3 row (0 none, 1 nodes 0/4 + midpoint,
// 2 all pairs + midpoint).
template <bool SMEM, bool CZ>
static const void *leaf2_src_kernel_l3(int l3s) {
    if (l3s == 2) return (const void *)k_leaf2_sym3<LEAF2_PPL3, SMEM, CZ, true, 2>;
    if (l3s == 1) return (const void *)k_leaf2_sym3<LEAF2_PPL3, SMEM, CZ, true, 1>;
    return (const void *)k_leaf2_sym3<LEAF2_PPL3, SMEM, CZ, true, 0>;
}
static const void *leaf2_src_kernel(bool smem, bool cz, int l3s) {
    return smem ? (cz ? leaf2_src_kernel_l3<true, true>(l3s) : leaf2_src_kernel_l3<true, false>(l3s))
                : (cz ? leaf2_src_kernel_l3<false, true>(l3s) : leaf2_src_kernel_l3<false, false>(l3s));
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
    // source tasks are only understood by k_leaf2_sym3 (plan.cpp builds them for that kernel alone)
    if (p->leaf2 && hp.leaf2_srctasks && !(p->cplx && sy && ct && nj == 3 && hp.leaf2_ppl >= 2))
        return SG_EUNSUPPORTED;
    if (hp.leaf2_groups > 1 && (p->cplx || hp.leaf2_ppl != 1)) return SG_EUNSUPPORTED;   // plan.cpp never does this
    const void *fn = p->leaf2 ? (p->cplx ? leaf2_kernel<true>(nj, sm, ct, sy, cz, hp.leaf2_ppl)
                                         : leaf2_kernel<false>(nj, sm, ct, sy, cz, 1, hp.leaf2_groups))
                              : (p->cplx ? leaf1_kernel<true>(nj, sm) : leaf1_kernel<false>(nj, sm));
    if (p->leaf1_smem > 48 * 1024 &&
        cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)p->leaf1_smem) != cudaSuccess)
        return SG_ECUDA;
    if (hp.leaf2_srctasks) {
        // exactly conjugate level-3 pairs (x_j = 1 - x_{4-j}, equal weights) and an exactly real
        // midpoint (x_2 = 1/2): shared products in the source tasks' level-3 rows
        const int e3 = hp.entry_off[3];
        auto pair = [&](int a, int b) {
            return 1.0 - hp.X[e3 + b] == hp.X[e3 + a] && hp.Whi[e3 + a] == hp.Whi[e3 + b] &&
                   hp.Wlo[e3 + a] == hp.Wlo[e3 + b];
        };
        const bool p04 = pair(0, 4) && hp.X[e3 + 2] == 0.5, p13 = pair(1, 3);
        p->leaf2_l3s = p04 ? (p13 ? 2 : 1) : 0;
#ifdef LEAF2_NO_L3SYM
        p->leaf2_l3s = 0;
#endif
    }
    if (hp.leaf2_srctasks && p->leaf1_smem > 48 * 1024 &&
        cudaFuncSetAttribute(leaf2_src_kernel(true, cz, p->leaf2_l3s), cudaFuncAttributeMaxDynamicSharedMemorySize,
                             (int)p->leaf1_smem) != cudaSuccess)
        return SG_ECUDA;
    // k_leaf2_sym3 has its own CTA size; every other leaf kernel runs PASS_THREADS
    p->leaf2_threads = (p->leaf2 && p->cplx && sy && ct && nj == 3 && hp.leaf2_ppl >= 2) ? SYM3_THREADS
                       : (p->leaf2 && !p->cplx)                                       ? LEAF2_REAL_THREADS
                       : p->leaf2                                                     ? PASS_THREADS
                                                                                      : LEAF1_THREADS;
    const int wpb = p->leaf2_threads / 32;
    int per_sm = 0, dev = 0, sms = 0;
    if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, fn, p->leaf2_threads, p->leaf1_smem) != cudaSuccess ||
        cudaGetDevice(&dev) != cudaSuccess ||
        cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess)
        return SG_ECUDA;
    const long long ntasks = hp.pass_ntasks[t];
    p->leaf1_grid = std::max<long long>(1, std::min<long long>((ntasks + wpb - 1) / wpb, (long long)sms * per_sm));
    p->resident_ctas = sms * per_sm;
    hp.pass_blocks[t] = ntasks;   // partial slots: one per task (0 tasks -> no slot, no launch)
    layout_partials(hp);
    p->leaf1_t = t;
    return SG_OK;
}

template <bool CPLX>
static void launch_leaf2(sg_plan_s *p, const Leaf2Args &A, int nj, cudaStream_t st) {
    const unsigned grid = (unsigned)p->leaf1_grid;
    const size_t sm = p->leaf1_smem;
    const void *fn = leaf2_kernel<CPLX>(nj, sm > 0, p->leaf2_center, p->leaf2_sym, p->leaf2_cz, p->hp.leaf2_ppl,
                                        p->hp.leaf2_groups);
    DevPlan dp = p->dp;
    Leaf2Args a = A;
    void *args[] = {&dp, &a};
    cudaLaunchKernel(fn, dim3(grid), dim3(p->leaf2_threads), args, sm, st);
}

static void launch_leaf2_src(sg_plan_s *p, const Leaf2Args &A, cudaStream_t st) {
    const size_t sm = p->leaf1_smem;
    const void *fn = leaf2_src_kernel(sm > 0, p->leaf2_cz, p->leaf2_l3s);
    const unsigned grid = (unsigned)std::min<long long>(p->leaf1_grid, A.ntasks);
    DevPlan dp = p->dp;
    Leaf2Args a = A;
    void *args[] = {&dp, &a};
    cudaLaunchKernel(fn, dim3(grid), dim3(SYM3_THREADS), args, sm, st);
}

template <bool CPLX>
static void launch_leaf1(sg_plan_s *p, const PassArgs &A, int nj, cudaStream_t st) {
    const unsigned grid = (unsigned)p->leaf1_grid;
    const size_t sm = p->leaf1_smem;
    if (nj == 3) {
        if (sm) k_leaf1<CPLX, 3, true><<<grid, LEAF1_THREADS, sm, st>>>(p->dp, A);
        else k_leaf1<CPLX, 3, false><<<grid, LEAF1_THREADS, 0, st>>>(p->dp, A);
    } else {
        if (sm) k_leaf1<CPLX, 2, true><<<grid, LEAF1_THREADS, sm, st>>>(p->dp, A);
        else k_leaf1<CPLX, 2, false><<<grid, LEAF1_THREADS, 0, st>>>(p->dp, A);
    }
}

// K0 / head launches, one instantiation per integrand kind (factor form: kinds 0-3)
static void launch_factor_base(const DevPlan &dp, int nfb, cudaStream_t st) {
    const unsigned g = (unsigned)(nfb + 1);
    switch (dp.kind) {
    case SG_F_EXP_LINEAR: k_factor_base<SG_F_EXP_LINEAR><<<g, K0_THREADS, 0, st>>>(dp, nfb); break;
    case SG_F_OSCILLATORY: k_factor_base<SG_F_OSCILLATORY><<<g, K0_THREADS, 0, st>>>(dp, nfb); break;
    case SG_F_PRODUCT_PEAK: k_factor_base<SG_F_PRODUCT_PEAK><<<g, K0_THREADS, 0, st>>>(dp, nfb); break;
    case SG_F_GAUSSIAN: k_factor_base<SG_F_GAUSSIAN><<<g, K0_THREADS, 0, st>>>(dp, nfb); break;
    }
}
static void launch_head(const DevPlan &dp, const RootArgs &R, unsigned grid, cudaStream_t st) {
    switch (dp.kind) {
    case SG_F_EXP_LINEAR: k_head<SG_F_EXP_LINEAR><<<grid, HEAD_THREADS, 0, st>>>(dp, R); break;
    case SG_F_OSCILLATORY: k_head<SG_F_OSCILLATORY><<<grid, HEAD_THREADS, 0, st>>>(dp, R); break;
    case SG_F_PRODUCT_PEAK: k_head<SG_F_PRODUCT_PEAK><<<grid, HEAD_THREADS, 0, st>>>(dp, R); break;
    case SG_F_GAUSSIAN: k_head<SG_F_GAUSSIAN><<<grid, HEAD_THREADS, 0, st>>>(dp, R); break;
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

// Profiling: sg_integrate records CUDA events (plan-owned) and, per launch, the pair (start event,
// end event) whose difference sg_profile_read reports.  Sequential launches chain (the end of one is
// the start of the next); the two concurrent passes (fork/join below) both start at the fork event.
struct ProfRec {
    sg_plan_s *p;
    cudaStream_t st;
    unsigned flags;
    int nev = 0;
    int last = -1;   // index of the most recent event on the main stream
    int rec(cudaStream_t on) {
        if (!p->prof || p->prof_mode == 2 || nev >= (int)p->ev.size()) return -1;
        cudaEventRecordWithFlags(p->ev[nev], on, flags);
        return nev++;
    }
    void launch_done(int start, int end) {
        if (p->prof) p->prof_pairs.push_back({start, end});
    }
    // mode 2 (sg_profile_enable(p, 2)): events around the dominant pass's launch only
    int dom_rec(cudaStream_t on, int t) {
        if (!p->prof || p->prof_mode != 2 || t != p->prof_dom || nev >= (int)p->ev.size()) return -1;
        cudaEventRecordWithFlags(p->ev[nev], on, flags);
        return nev++;
    }
    // a sequential launch just issued on the main stream
    void seq() {
        const int e = rec(st);
        launch_done(last, e);
        last = e;
    }
};

extern "C" int sg_integrate(sg_plan_t p, sg_stream_t s, double *out_dev) {
    if (!p || !out_dev) return SG_EINVAL;
    if (!p->ws) return SG_ENOWORKSPACE;
    cudaStream_t st = (cudaStream_t)s;
    const HostPlan &hp = p->hp;
    const DevPlan &dp = p->dp;
    double2 *partials = (double2 *)(p->ws + p->ws_part_off);
    // under stream capture the events become graph event-record nodes (timed on every replay)
    cudaStreamCaptureStatus cap = cudaStreamCaptureStatusNone;
    if (p->prof && cudaStreamIsCapturing(st, &cap) != cudaSuccess) return SG_ECUDA;
    ProfRec pr{p, st, cap == cudaStreamCaptureStatusActive ? (unsigned)cudaEventRecordExternal : 0u};
    p->prof_pairs.clear();
    pr.last = pr.rec(st);
    const int nfb = (int)((hp.tab_entries + K0_THREADS - 1) / K0_THREADS);   // factor-table blocks of the merged K0 launch
    if (p->plain || p->collapse) {
        // status words: these paths' final kernels also close the step (step_close_status)
        launch_factor_base(dp, nfb, st);
        pr.seq();
        pr.launch_done(pr.last, pr.last);   // K0 base: merged into the factor launch
    }
    if (p->plain) {
        double2 *part = (double2 *)(p->ws + p->ws_part_off);
        k_plain<<<p->plain_blocks, 256, 0, st>>>(dp, p->utabs, part);
        pr.seq();
        k_reduce<<<1, 1024, 0, st>>>(dp, part, p->plain_blocks, 0, out_dev);
        pr.seq();
        if (cudaGetLastError() != cudaSuccess) return SG_ECUDA;
        return SG_OK;
    }
    if (p->collapse) {
        const int L = hp.L;
        double2 *pre = (double2 *)(p->ws + p->ws_part_off);
        double2 *pim = pre + (size_t)p->collapse_blocks * (L + 1);
        const size_t smem_part = (size_t)(p->cplx ? 4 : 2) * COLLAPSE_THREADS * (L + 1) * sizeof(double2);
        const size_t smem_fin = (size_t)(p->cplx ? 2 : 1) * COLLAPSE_THREADS * (L + 1) * sizeof(double2);
        if (p->cplx) {
            k_collapse_part<true><<<p->collapse_blocks, COLLAPSE_THREADS, smem_part, st>>>(dp, pre, pim);
            pr.seq();
            k_collapse_final<true><<<1, COLLAPSE_THREADS, smem_fin, st>>>(dp, pre, pim, p->collapse_blocks,
                                                                         p->collapse_emit ? 1 : 0, out_dev);
        } else {
            k_collapse_part<false><<<p->collapse_blocks, COLLAPSE_THREADS, smem_part, st>>>(dp, pre, pim);
            pr.seq();
            k_collapse_final<false><<<1, COLLAPSE_THREADS, smem_fin, st>>>(dp, pre, pim, p->collapse_blocks,
                                                                          p->collapse_emit ? 1 : 0, out_dev);
        }
        pr.seq();
        if (cudaGetLastError() != cudaSuccess) return SG_ECUDA;
        return SG_OK;
    }
    // Task counters (plan-owned, zero at the start of every step; re-armed by k_reduce_fused):
    // [0] the persistent last-pass kernel, [1] the reduction ticket, [2] the source-task kernel.
    unsigned long long *cnt_leaf = p->d_counter, *cnt_src = p->d_counter + 2;
    RootArgs R;
    memset(&R, 0, sizeof R);
    R.lo = hp.range_lo;
    R.hi = hp.range_hi;
    R.off1 = p->d_tabs + p->tab_off1;
    R.JS = p->d_tabs + p->tab_JS;
    if (hp.nfront >= 1) front_ptrs(p, 1, R.dst_re, R.dst_im, R.dst_meta);
    R.partials = partials;
#ifdef SG_CHECKS
    R.chk_src_cap = 0;
    R.chk_dst_cap = hp.ws_front_cap[1];
#endif
    if (p->head) {
        // K0 + base + root pass + analytic suffix bounds in one launch (k_head, k_factor.cuh)
        launch_head(dp, R, (unsigned)hp.root_blocks, st);
        pr.seq();
        pr.launch_done(pr.last, pr.last);   // K0 base: merged
        pr.launch_done(pr.last, pr.last);   // root pass: merged
    } else {
        // K0 (factor table + base), then the suffix bounds of |F|
        if (p->sform) {
            if (p->sform_dd) k_factor_base_s<true><<<nfb + 1, K0_THREADS, 0, st>>>(dp, nfb);
            else k_factor_base_s<false><<<nfb + 1, K0_THREADS, 0, st>>>(dp, nfb);
        } else {
            launch_factor_base(dp, nfb, st);
            if (hp.tab_entries > 0) k_suffix_abs<<<hp.L, SUFFIX_THREADS, 0, st>>>(dp);
        }
        pr.seq();
        pr.launch_done(pr.last, pr.last);   // K0 base: merged into the factor launch
        // root pass
        if (p->sform)
            (p->sform_dd ? k_root_s<true> : k_root_s<false>)<<<(unsigned)hp.root_blocks, 256, 0, st>>>(dp, R);
        else if (p->cplx)
            k_root<true><<<(unsigned)hp.root_blocks, 256, 0, st>>>(dp, R);
        else
            k_root<false><<<(unsigned)hp.root_blocks, 256, 0, st>>>(dp, R);
        pr.seq();
    }
    // Fused plans: pass nfront-1 writes no frontier (its children are the fused kernel's business),
    // so it and the fused pass nfront both only read frontier nfront-1 — they run concurrently, pass
    // nfront-1 on the plan's side stream (fork/join through events; graph branches under capture).
    // The persistent fused kernel takes the SMs the shorter pass leaves or frees (its tail fill).
    // passes nfront-1 || nfront on shards of a world (their tails matter); at world 1 only when the
    // fused grid leaves SMs free (fork1: configs 1-2); otherwise the fused pass runs alone (same step
    // time within 0.2% on configs 4-5, and a clean kernel interval)
    const bool fork = p->leaf2 && p->side != nullptr && hp.nfront >= 2 && (p->world > 1 || p->fork1);
    int ev_fork = -1;
    // level-synchronous passes
    for (int t = 1; t <= hp.nfront; ++t) {
        cudaStream_t sx = st;
        bool split_done = false;
        if (fork && t == hp.nfront - 1) {
            if (cudaEventRecord(p->ev_fork, st) != cudaSuccess) return SG_ECUDA;
            if (cudaStreamWaitEvent(p->side, p->ev_fork, 0) != cudaSuccess) return SG_ECUDA;
            ev_fork = pr.last;
            sx = p->side;
        }
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
            B.counter = cnt_leaf;
            B.prefetch = B.ntasks >= (long long)p->prefetch_min * p->leaf1_grid * (p->leaf2_threads / 32) ? 1 : 0;
#ifdef SG_CHECKS
            B.chk_src_cap = hp.ws_front_cap[(t - 1) % 2];
            B.chk_dst_cap = 0;
#endif
            const int d0 = pr.dom_rec(st, t);
            if (B.ntasks > 0) {
                if (p->cplx) launch_leaf2<true>(p, B, hp.nl[2], st);
                else launch_leaf2<false>(p, B, hp.nl[2], st);
            }
            const int d1 = pr.dom_rec(st, t);
            if (p->prof_mode == 2) {
                pr.launch_done(d0, d1);
            } else if (fork) {
                const int e = pr.rec(st);
                pr.launch_done(ev_fork, e);
                pr.last = e;
            } else {
                pr.seq();
            }
            continue;
        }
        const int d0 = pr.dom_rec(sx, t);
        if (hp.leaf2_srctasks && p->leaf2 && t == hp.nfront - 1) {
            // pass L-2 as k_leaf2_sym3 source tasks over every source of frontier L-2
            Leaf2Args S;
            memset(&S, 0, sizeof S);
            double2 *re, *im;
            uint32_t *meta;
            front_ptrs(p, t, re, im, meta);
            S.src_re = re;
            S.src_im = im;
            S.T2 = p->d_tabs + p->tab_TKS;
            S.ntasks = hp.pass_ntasks[t];
            S.partials = partials + hp.pass_partial_off[t];
            S.counter = cnt_src;
            S.prefetch = 0;
#ifdef SG_CHECKS
            S.chk_src_cap = hp.ws_front_cap[t % 2];
            S.chk_dst_cap = 0;
#endif
            if (S.ntasks > 0) launch_leaf2_src(p, S, sx);
        } else {
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
            A.counter = cnt_leaf;   // k_leaf1 (the last pass of an unfused plan)
#ifdef SG_CHECKS
            A.chk_src_cap = hp.ws_front_cap[t % 2];
            A.chk_dst_cap = write ? hp.ws_front_cap[(t + 1) % 2] : 0;
#endif
            const unsigned grid = (unsigned)hp.pass_blocks[t];
            size_t pass_smem = 0;
            if (write && !p->sform) {
                // stage factor levels 2 .. while they fit p->pass_smem_cap bytes (k_pass)
                const size_t per = p->cplx ? 2 * sizeof(double2) : sizeof(double2);
                int lmax = 1, ent = 0;
                for (int l = 2; l <= hp.L + 1; ++l) {
                    const int e = hp.d * hp.nl[l];
                    if ((size_t)(ent + e) * per > p->pass_smem_cap) break;
                    ent += e;
                    lmax = l;
                }
                A.stage_lmax = lmax >= 2 ? lmax : 0;
                A.stage_entries = ent;
                pass_smem = (size_t)ent * per;
            }
            // single-level last pass (every source has excess L-1): specialised k_leaf1
            const int n2 = hp.nl[2];
            const bool single = !write && t == p->leaf1_t;
            if (p->sform) {
                if (p->sform_dd) {
                    if (write) k_pass_s<true, true><<<grid, PASS_THREADS, 0, sx>>>(dp, A);
                    else k_pass_s<true, false><<<grid, PASS_THREADS, 0, sx>>>(dp, A);
                } else {
                    if (write) k_pass_s<false, true><<<grid, PASS_THREADS, 0, sx>>>(dp, A);
                    else k_pass_s<false, false><<<grid, PASS_THREADS, 0, sx>>>(dp, A);
                }
            } else if (write && hp.pass_split[t] && p->side != nullptr) {
                // split frontier pass: write-only k_pass here, leaf-only k_leaf on the side stream
                // (both read frontier t; partial slots [0, grid) and [grid, 2 grid) of the pass)
                PassArgs A2 = A;
                A2.dst_re = A2.dst_im = nullptr;
                A2.dst_meta = nullptr;
                A2.TB = nullptr;
                A2.partials = A.partials + hp.pass_front_slots[t];
                A.counter = p->d_counter + 4;   // k_front's chunk counter (zeroed per split pass)
                if (cudaMemsetAsync(A.counter, 0, sizeof(unsigned long long), st) != cudaSuccess) return SG_ECUDA;
#ifdef SG_CHECKS
                A2.chk_dst_cap = 0;
#endif
                if (cudaEventRecord(p->ev_fork, st) != cudaSuccess) return SG_ECUDA;
                if (cudaStreamWaitEvent(p->side, p->ev_fork, 0) != cudaSuccess) return SG_ECUDA;
                const FrontChunk *runs = p->d_runs + p->runs_off[t];
                const long long nr = p->runs_n[t];
                // profile entry of the pass = k_front (fork -> its end on this stream).  Concurrent
                // (default): the leaf-only k_leaf overlaps it on the side stream.  Serial
                // (SG_B200_SPLIT_SERIAL=1: the clean frontier-kernel time of bench.py's frontier leg):
                // k_leaf follows on this stream and falls into the next launch's interval.
                if (!p->split_serial) {
                    if (p->cplx) k_leaf<true, true><<<grid, PASS_THREADS, 0, p->side>>>(dp, A2);
                    else k_leaf<false, true><<<grid, PASS_THREADS, 0, p->side>>>(dp, A2);
                }
                if (p->cplx) k_front<true><<<p->front_grid, FRONT_THREADS, 0, st>>>(dp, A, runs, nr);
                else k_front<false><<<p->front_grid, FRONT_THREADS, 0, st>>>(dp, A, runs, nr);
                split_done = true;
                if (p->prof_mode != 2) {
                    const int e = pr.rec(st);
                    pr.launch_done(pr.last, e);
                    pr.last = e;
                }
                if (p->split_serial) {
                    if (p->cplx) k_leaf<true, true><<<grid, PASS_THREADS, 0, st>>>(dp, A2);
                    else k_leaf<false, true><<<grid, PASS_THREADS, 0, st>>>(dp, A2);
                }
                if (cudaEventRecord(p->ev_join, p->side) != cudaSuccess) return SG_ECUDA;
                if (cudaStreamWaitEvent(st, p->ev_join, 0) != cudaSuccess) return SG_ECUDA;
            } else if (p->cplx) {
                if (write) k_pass<true, true><<<grid, PASS_THREADS, pass_smem, sx>>>(dp, A);
                else if (single) { if (A.ntasks > 0) launch_leaf1<true>(p, A, n2, sx); }
                else k_leaf<true><<<grid, PASS_THREADS, 0, sx>>>(dp, A);
            } else {
                if (write) k_pass<false, true><<<grid, PASS_THREADS, pass_smem, sx>>>(dp, A);
                else if (single) { if (A.ntasks > 0) launch_leaf1<false>(p, A, n2, sx); }
                else k_leaf<false><<<grid, PASS_THREADS, 0, sx>>>(dp, A);
            }
        }
        const int d1 = pr.dom_rec(sx, t);
        if (sx != st) {
            if (p->prof_mode == 2) pr.launch_done(d0, d1);
            else pr.launch_done(ev_fork, pr.rec(sx));
            if (cudaEventRecord(p->ev_join, sx) != cudaSuccess) return SG_ECUDA;
        } else if (p->prof_mode == 2) {
            pr.launch_done(d0, d1);
        } else if (!split_done) {
            pr.seq();
        }
    }
    if (fork && cudaStreamWaitEvent(st, p->ev_join, 0) != cudaSuccess) return SG_ECUDA;
    {
        const long long nl1 = std::max<long long>(1, (hp.total_partials + RED_CHUNK2 - 1) / RED_CHUNK2);
        double2 *l1 = (double2 *)(p->ws + p->ws_red_off);
        auto red = dp.sform == 2 ? k_reduce_fused<2> : dp.sform == 1 ? k_reduce_fused<1> : k_reduce_fused<0>;
        red<<<(unsigned)nl1, RED_THREADS, 0, st>>>(dp, partials, hp.total_partials, hp.include_root ? 1 : 0, out_dev,
                                                  l1, p->d_counter + 1, p->d_counter);
    }
    {
        // the reduction starts when both branches are done: time it from the later of the two ends
        const int e = pr.rec(st);
        pr.launch_done(pr.last, e);
    }
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
    int v = 0;   // status[1]: the flag of the last completed sg_integrate (k_finalize reads the same)
    if (cudaMemcpy(&v, p->dp.status + 1, sizeof(int), cudaMemcpyDeviceToHost) != cudaSuccess) return SG_ECUDA;
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
    const int n = (p->collapse || p->plain) ? 0 : p->hp.nfront + 1;   // no tree passes run
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
    if (!p || enable < 0 || enable > 2) return SG_EINVAL;
    p->prof_mode = enable;
    if (enable && p->ev.empty()) {
        p->ev.resize(6 + p->hp.nfront);
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
    const int nl = (p->collapse || p->plain) ? 4 : 4 + p->hp.nfront;
    if (!ms) {
        *n = nl;
        return SG_OK;
    }
    if (*n < nl || p->ev.empty() || (int)p->prof_pairs.size() != nl) return SG_EINVAL;
    for (int i = 0; i < nl; ++i) {
        const int a = p->prof_pairs[i].first, b = p->prof_pairs[i].second;
        if (a < 0 || b < 0 || a == b) {   // merged launch, or not timed (mode 2: only the dominant pass)
            ms[i] = 0.0f;
            continue;
        }
        if (cudaEventSynchronize(p->ev[b]) != cudaSuccess) return SG_ECUDA;
        if (cudaEventElapsedTime(&ms[i], p->ev[a], p->ev[b]) != cudaSuccess) return SG_ECUDA;
    }
    *n = nl;
    return SG_OK;
}

static int build_unrank_tables(sg_plan_s *p) {
    const HostPlan &hp = p->hp;
    if (!p->d_unrank) {
        const int d = hp.d, L = hp.L, W = d + 1;
        std::vector<unsigned long long> SG((size_t)(L + 1) * W, 0);
        auto sub = [&](int b, int k) -> unsigned long long { return hp.Sub[(size_t)b * W + (k + 1)]; };
        for (int b = 0; b <= L; ++b)
            for (int k = d - 1; k >= 0; --k) {
                unsigned long long g = 0;
                for (int lp = 2; lp <= L + 1 - b; ++lp) g += (unsigned long long)hp.nl[lp] * sub(b + lp - 1, k);
                SG[(size_t)b * W + k] = SG[(size_t)b * W + k + 1] + g;
            }
        const long long n1 = hp.range_hi - hp.range_lo;
        std::vector<unsigned long long> D1((size_t)n1 + 1, 0);
        for (long long i = 0; i < n1; ++i) {
            const long long r1 = hp.range_lo + i;
            const int k1 = (int)(r1 / hp.M0);
            int rem = (int)(r1 - (long long)k1 * hp.M0), l1 = 2;
            while (rem >= hp.nl[l1]) {
                rem -= hp.nl[l1];
                ++l1;
            }
            D1[(size_t)i + 1] = D1[(size_t)i] + sub(l1 - 1, k1);
        }
        const size_t nsub = hp.Sub.size(), nsg = SG.size(), nd1 = D1.size();
        if (cudaMalloc(&p->d_unrank, sizeof(unsigned long long) * (nsub + nsg + nd1)) != cudaSuccess) {
            cudaGetLastError();
            p->d_unrank = nullptr;
            return SG_ENOMEM;
        }
        unsigned long long *q = (unsigned long long *)p->d_unrank;
        bool ok = cudaMemcpy(q, hp.Sub.data(), sizeof(unsigned long long) * nsub, cudaMemcpyHostToDevice) == cudaSuccess;
        ok &= cudaMemcpy(q + nsub, SG.data(), sizeof(unsigned long long) * nsg, cudaMemcpyHostToDevice) == cudaSuccess;
        ok &= cudaMemcpy(q + nsub + nsg, D1.data(), sizeof(unsigned long long) * nd1, cudaMemcpyHostToDevice) == cudaSuccess;
        if (!ok) return SG_ECUDA;
        p->utabs.Sub = q;
        p->utabs.SG = q + nsub;
        p->utabs.D1 = q + nsub + nsg;
        p->utabs.lo = hp.range_lo;
        p->utabs.n1 = n1;
        p->utabs.include_root = hp.include_root ? 1 : 0;
        p->utabs.merge = hp.merge;
        p->utabs.shard_points = hp.shard_points;
    }
    return SG_OK;
}

extern "C" int sg_eval_points(sg_plan_t p, sg_stream_t s, const unsigned long long *index_dev, long long n,
                              int *points_dev, double *terms_dev) {
    if (!p || n < 0 || (n > 0 && (!index_dev || !points_dev || !terms_dev))) return SG_EINVAL;
    if (p->sform || p->collapse) return SG_EUNSUPPORTED;
    cudaStream_t st = (cudaStream_t)s;
    const HostPlan &hp = p->hp;
    int rc = build_unrank_tables(p);
    if (rc) return rc;
    // the factor table and base of the current parameters (K0), then one thread per index
    const int nfb = (int)((hp.tab_entries + K0_THREADS - 1) / K0_THREADS);
    launch_factor_base(p->dp, nfb, st);
    if (n > 0)
        k_eval_points<<<(unsigned)((n + 127) / 128), 128, 0, st>>>(p->dp, p->utabs, index_dev, n, points_dev,
                                                                   terms_dev);
    // keep the invariant "status[0] is clear when a step starts" (non-finite factors show as NaN terms)
    if (cudaMemsetAsync(p->dp.status, 0, sizeof(int), st) != cudaSuccess) return SG_ECUDA;
    if (cudaGetLastError() != cudaSuccess) return SG_ECUDA;
    return SG_OK;
}

#ifdef SG_CHECKS
// Checked build only (not in include/sg_b200.h): arm the checks for the next sg_integrate / read them.
static unsigned *g_chk_writes_host = nullptr;
static long long g_chk_writes_cap = 0;
extern "C" int sg_chk_begin(sg_plan_t p) {
    if (!p || !p->ws) return SG_EINVAL;
    const long long n = p->collapse ? 0 : p->plain ? p->plain_blocks : p->hp.total_partials;
    if (n > g_chk_writes_cap) {
        if (g_chk_writes_host) cudaFree(g_chk_writes_host);
        if (cudaMalloc(&g_chk_writes_host, sizeof(unsigned) * (size_t)n) != cudaSuccess) return SG_ENOMEM;
        g_chk_writes_cap = n;
    }
    if (n > 0 && cudaMemset(g_chk_writes_host, 0, sizeof(unsigned) * (size_t)n) != cudaSuccess) return SG_ECUDA;
    ChkState st;
    memset(&st, 0, sizeof st);
    st.writes = g_chk_writes_host;
    st.nslots = n;
    st.part_base = (const double2 *)(p->ws + p->ws_part_off);
    if (cudaMemcpyToSymbol(g_chk, &st, sizeof st) != cudaSuccess) return SG_ECUDA;
    return SG_OK;
}
// out[0] = violations, out[1..4] = first (code, index, bound, line), out[5] = slots not written exactly
// once, out[6] = slots checked
extern "C" int sg_chk_end(sg_plan_t p, long long *out) {
    if (!p || !out) return SG_EINVAL;
    if (cudaDeviceSynchronize() != cudaSuccess) return SG_ECUDA;
    ChkState st;
    if (cudaMemcpyFromSymbol(&st, g_chk, sizeof st) != cudaSuccess) return SG_ECUDA;
    std::vector<unsigned> w((size_t)st.nslots);
    if (st.nslots > 0 && cudaMemcpy(w.data(), st.writes, sizeof(unsigned) * (size_t)st.nslots,
                                    cudaMemcpyDeviceToHost) != cudaSuccess)
        return SG_ECUDA;
    long long bad = 0;
    for (unsigned v : w) bad += (v != 1);
    out[0] = (long long)st.viol;
    for (int i = 0; i < 4; ++i) out[1 + i] = st.first[i];
    out[5] = bad;
    out[6] = st.nslots;
    return SG_OK;
}
#endif

#ifdef SG_TAILPROF
// experiment build only: copy the per-warp records of the last k_leaf2 launch (n <= TAILPROF_MAX)
extern "C" int sg_tailprof_reset() {
    static unsigned long long z[TAILPROF_MAX];
    if (cudaMemcpyToSymbol(g_tp_t0, z, sizeof z) != cudaSuccess || cudaMemcpyToSymbol(g_tp_t1, z, sizeof z) != cudaSuccess)
        return SG_ECUDA;
    return SG_OK;
}
extern "C" int sg_tailprof_read(unsigned long long *t0, unsigned long long *t1, unsigned *sm, unsigned *ntask,
                                unsigned *kmids, int n) {
    if (n > TAILPROF_MAX || cudaDeviceSynchronize() != cudaSuccess) return SG_EINVAL;
    if (cudaMemcpyFromSymbol(t0, g_tp_t0, sizeof(unsigned long long) * n) != cudaSuccess ||
        cudaMemcpyFromSymbol(t1, g_tp_t1, sizeof(unsigned long long) * n) != cudaSuccess ||
        cudaMemcpyFromSymbol(sm, g_tp_sm, sizeof(unsigned) * n) != cudaSuccess ||
        cudaMemcpyFromSymbol(ntask, g_tp_n, sizeof(unsigned) * n) != cudaSuccess ||
        cudaMemcpyFromSymbol(kmids, g_tp_rows, sizeof(unsigned) * n) != cudaSuccess)
        return SG_ECUDA;
    return SG_OK;
}
#endif

extern "C" int sg_destroy(sg_plan_t p) {
    if (!p) return SG_EINVAL;
    for (auto &e : p->ev) cudaEventDestroy(e);
    if (p->ev_fork) cudaEventDestroy(p->ev_fork);
    if (p->ev_join) cudaEventDestroy(p->ev_join);
    if (p->side) cudaStreamDestroy(p->side);
    if (p->d_runs) cudaFree(p->d_runs);
    if (p->d_unrank) cudaFree(p->d_unrank);
    if (p->dev_block) cudaFree(p->dev_block);
    delete p;
    return SG_OK;
}
