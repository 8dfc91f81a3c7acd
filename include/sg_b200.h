/*
 * sg_b200.h — C ABI of the B200 Smolyak sparse-grid quadrature hot path (arXiv 2210.14313, MDI-SG).
 *
 * The library evaluates the Smolyak combination sum (Eq 2.6; tensor rule
 * PAPER.md:69-71, Eq 2.7) on the unit cube [0,1]^d (reading R2 of DESIGN.md):
 *
 *   A(q,d) f = sum_{q-d+1 <= |i| <= q} (-1)^{q-|i|} C(d-1, q-|i|) (U^{i_1} x ... x U^{i_d}) f
 *
 * with q = d + L, by the paper's multilevel dimension iteration (Eqs 3.8-3.11):
 * points sharing a prefix of active coordinates share one partial result, carried one active
 * coordinate at a time through a level-synchronous prefix tree on the GPU.  Every Smolyak point
 * (the n_d^q of PAPER.md:73-75) is evaluated individually; no point list is ever stored.
 *
 * Conventions for every entry point:
 *  - Return value: SG_OK (0) or a negative sg_status code; no C++ exception crosses the ABI.
 *  - "host" pointers are ordinary CPU memory; "device" pointers are CUDA global memory of the
 *    current device.  The library never frees caller memory.
 *  - Asynchronous entry points only ENQUEUE work on the given stream; the caller synchronises.
 *  - A plan is immutable after sg_plan (except sg_update_integrand / sg_set_workspace) and may be
 *    used by one stream at a time.
 */
#ifndef SG_B200_H
#define SG_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct CUstream_st *sg_stream_t;  /* == cudaStream_t; NULL = legacy default stream */

/* Status codes (error vocabulary after SPEC.md:66, 170, 194, 347). */
typedef enum {
    SG_OK = 0,
    SG_EINVAL = -1,        /* d < 1, q < d (BudgetTooSmall), NULL pointer, bad enum, non-finite
                              parameter, w missing for peak/gauss, rank/world/range inconsistent */
    SG_EUNSUPPORTED = -2,  /* UnsupportedLevel: CC max level L+1 > 12 (its weights cost O(n^2) quad
                              cosines at plan time), trapezoidal L+1 > 20, GL n > 64,
                              Gauss-Patterson rule > 63 points, d > 2^20-1, L > 19 */
    SG_EOVERFLOW = -3,     /* a point or frontier count would reach 2^63 */
    SG_ENOMEM = -4,        /* device allocation failed, or workspace smaller than required */
    SG_ECUDA = -5,         /* a CUDA runtime call failed (launch error, bad stream, ...) */
    SG_ENONFINITE = -6,    /* NonFiniteIntegrand: a per-coordinate factor or the result is not
                              finite; the result is NaN */
    SG_ENOWORKSPACE = -7   /* sg_integrate called before sg_set_workspace */
} sg_status;

/* 1-D rule families, numbered by the paper's parameter r. */
typedef enum {
    SG_RULE_TRAPEZOIDAL = 1,      /* nested, n_1 = 1, n_l = 2^{l-1}+1, equal spacing, end weights
                                     halved (Eq 2.10)                          */
    SG_RULE_CLENSHAW_CURTIS = 2,  /* nested, n_1 = 1, n_l = 2^{l-1}+1 (Eq 2.11) */
    SG_RULE_GAUSS_PATTERSON = 3,  /* nested, delayed: n_l = 1, 3, 3, 7, 7, 7, 15, ... = the smallest
                                     Patterson rule exact to degree 2l-1 (Eq 2.12,
                                     sequence of PAPER.md:615; reading R16)            */
    SG_RULE_GAUSS_LEGENDRE = 4    /* n_l = l (Eq 2.13)                         */
} sg_rule;

/* Integrand kinds (BASELINE.json configs; Genz families).  Kinds 0-3 are products of
 * per-coordinate factors (or the real part of one), which the MDI prefix tree carries as partial
 * products.  Kind 4 is not: the tree carries the partial sum s = sum_k c_k x_k and the outer
 * function is applied once per point (SG_ARITH_SFORM_DD). */
typedef enum {
    SG_F_EXP_LINEAR = 0,    /* f(x) = exp(sum_k c_k x_k)                                      */
    SG_F_OSCILLATORY = 1,   /* f(x) = cos(2 pi u + sum_k c_k x_k)                              */
    SG_F_PRODUCT_PEAK = 2,  /* f(x) = prod_k (c_k^-2 + (x_k - w_k)^2)^-1                        */
    SG_F_GAUSSIAN = 3,      /* f(x) = exp(-sum_k c_k^2 (x_k - w_k)^2)                           */
    SG_F_CORNER_PEAK = 4    /* f(x) = (1 + sum_k c_k x_k)^-(d+1), requires 1 + sum min(c_k,0) > 0
                               (SG_EINVAL at sg_plan; sg_update_integrand values outside the
                               domain set the NonFiniteIntegrand flag) */
} sg_kind;

/* Integrand description.  c: host array of d doubles (required); w: host array of d doubles
 * (required for PRODUCT_PEAK and GAUSSIAN, ignored otherwise); u: phase (OSCILLATORY only).
 * Copied by sg_plan / sg_update_integrand; the caller keeps ownership. */
typedef struct {
    sg_kind kind;
    int d;
    const double *c;
    const double *w;
    double u;
} sg_integrand_desc;

/* Form of the sum.  COMBINATION = literal Eq 2.6 (coefficients (-1)^{L-e} C(d-1, L-e) on the band
 * e >= L-d+1); DELTA = the coordinate-wise difference form that Eq 2.9 stands for (reading R6):
 * sum_{e=0}^{L} sum_{|i|=d+e} (Delta^{i_1} x ... x Delta^{i_d}) f, coefficient 1.  Same value. */
typedef enum { SG_FORM_COMBINATION = 0, SG_FORM_DELTA = 1 } sg_form;

/* Leaf arithmetic.
 *  FACTOR_DD  = double-double partial products of plan-time per-(coordinate,node) factors
 *               (parity-grade, default; kinds 0-3).  For SG_F_CORNER_PEAK, which has no factor
 *               form, FACTOR_DD selects SFORM_DD.
 *  SFORM_FP64 = ablation: FP64 partial sums of the argument and per-point FP64 exp/cos/pow (not
 *               parity-grade on ill-conditioned problems).
 *  SFORM_DD   = double-double partial sums of the argument and a per-point dd outer function
 *               (exp, cos, or the corner peak's power): parity-grade, ~20-40x the FP64 work of the
 *               factor form per point; the general path for non-separable outer functions.
 * The s-forms support kinds EXP_LINEAR, OSCILLATORY, GAUSSIAN and CORNER_PEAK (PRODUCT_PEAK ->
 * SG_EUNSUPPORTED), the tree method only, no merge (SG_EUNSUPPORTED). */
typedef enum { SG_ARITH_FACTOR_DD = 0, SG_ARITH_SFORM_FP64 = 1, SG_ARITH_SFORM_DD = 2 } sg_arith;

/* Repeated-point merging (Eq 2.8 writes Q as one weighted sum over the points, and
 * the Fig 2.1 remark: "we would avoid the repeated points").  Every level of a rule that contains
 * the midpoint 1/2 repeats it, and a point with a coordinate at 1/2 is the same point whether that
 * coordinate is at level 1 or at a higher level.
 *  MERGE_NONE     = every Eq 2.6/2.7 point is evaluated (n_d^q points).
 *  MERGE_MIDPOINT = the tree only carries non-midpoint nodes; all the copies of a point that differ
 *                   in the levels of its midpoint coordinates are summed into one merged
 *                   coefficient C'(t, b) = sum_{e=b}^{L} c(e) [z^{e-b}] M(z)^{d-t}
 *                   (t = non-midpoint actives, b = their excess, M(z) = 1 + sum_{l>=2} w^l(1/2) z^{l-1}
 *                   the midpoint's weights per level; c(e) the form's coefficient), so each such
 *                   point is evaluated once.  Same value (an exact regrouping of Eq 2.6); the point
 *                   count is the number of tree nodes (sg_plan_points), 5x fewer on config 5.
 *                   Requires arith FACTOR_DD (else SG_EUNSUPPORTED). */
typedef enum { SG_MERGE_NONE = 0, SG_MERGE_MIDPOINT = 1 } sg_merge;

/* Evaluation method.
 *  METHOD_TREE     = the multilevel dimension iteration over the Smolyak points (default; every
 *                    point of the prefix tree is evaluated).
 *  METHOD_COLLAPSE = separable collapse: the paper's symbolic partial function f_{t-m}
 *                     carried as a truncated polynomial in the level budget.
 *                    All four kinds are Re(B prod_k E_k(x_k)), so the Eq 2.6 sum over every tensor
 *                    point of every multi-index of excess e is [z^e] prod_k p_k(z) with
 *                    p_k(z) = sum_{l=1}^{L+1} (sum_j w_j^l E_k(x_j^l)) z^{l-1}; A = Re(B sum_e
 *                    coef[e] [z^e] prod_k p_k).  O(d L^2) double-double work, no points; same value
 *                    as the tree up to dd rounding.  Not sharded: rank 0 of `world` emits the value,
 *                    every other rank a zero partial (so sg_finalize's sum is the value).  Requires
 *                    SG_MERGE_NONE (else SG_EINVAL) and SG_ARITH_FACTOR_DD (else SG_EUNSUPPORTED);
 *                    sg_plan_passes reports 0 passes. */
/*  METHOD_PLAIN    = opt-in ablation, not part of the hot path: the paper's plain SG comparison
 *                    system (SURVEY.md §2a P25 marks it out of scope), kept only to
 *                    measure what the MDI reuse saves (bench.py --plain-ablation; off by default)
 *                    on the GPU — no dimension iteration; every
 *                    point of the shard is unranked (device K1) and its term formed from its t
 *                    factors on its own (sg_eval_points' arithmetic), dd accumulation in a fixed
 *                    order.  Same value; measures what the MDI prefix reuse saves.  Factor
 *                    arithmetic only (else SG_EUNSUPPORTED); sg_plan_passes reports 0 passes;
 *                    profiling launches [K0 factor, K0 base, k_plain, k_reduce]. */
typedef enum { SG_METHOD_TREE = 0, SG_METHOD_COLLAPSE = 1, SG_METHOD_PLAIN = 2 } sg_method;

/* Work partition.  The Smolyak points are split into the root (all-midpoint point) and the
 * subtrees of the depth-1 prefixes (k1, l1, j1) = (first active coordinate, its level >= 2, its node),
 * ranked lexicographically: r1 = k1 * M0 + sum_{2<=l<l1} n_l + j1, M0 = sum_{l=2}^{L+1} n_l.
 * If range_hi > range_lo >= 0 this plan evaluates exactly the subtrees r1 in [range_lo, range_hi)
 * (plus the root iff range_lo == 0).  Otherwise it evaluates shard `rank` of `world` contiguous
 * ranges balanced by subtree point counts (root on rank 0).  NULL options = whole problem. */
typedef struct {
    sg_form form;
    sg_arith arith;
    int rank, world;
    long long range_lo, range_hi;
    sg_merge merge;   /* SG_MERGE_NONE (default) or SG_MERGE_MIDPOINT */
    sg_method method; /* SG_METHOD_TREE (default), SG_METHOD_COLLAPSE or SG_METHOD_PLAIN */
} sg_options;

typedef struct sg_plan_s *sg_plan_t;

/* Defined by: the problem Q_d^q(f) of PAPER.md:65-67 (Eq 2.6, accuracy level q, d dimensions) with
 * the tensor rules of PAPER.md:69-71 (Eq 2.7) and the 1-D rules of PAPER.md:103-147 (Eqs 2.10-2.13);
 * errors after SPEC.md:66 (UnsupportedLevel), 194 (Overflow), 347 (BudgetTooSmall).
 * Build a plan: validates arguments, builds the 1-D rule tables (double, correctly rounded from
 * quad evaluations of Eqs 2.11/2.13 on [0,1]), the counting tables of the prefix tree and the
 * shard range; allocates plan-owned device tables and copies the integrand parameters (H2D,
 * synchronous).  q = d + L.  On success *out owns device memory until sg_destroy. */
int sg_plan(int d, int q, sg_rule rule, const sg_integrand_desc *f, const sg_options *opt,
            sg_plan_t *out);

/* Defined by: DESIGN.md §5 (no paper passage: the frontier of the level-synchronous walk of
 * PAPER.md:248-295 needs scratch that the caller owns).
 * Bytes of caller-provided device workspace (frontier ping-pong buffers + reduction partials). */
int sg_workspace_size(sg_plan_t p, size_t *bytes);

/* Defined by: DESIGN.md §5 (ownership contract of SURVEY.md §8b).
 * Attach caller-owned device workspace of at least sg_workspace_size bytes (256-byte aligned). */
int sg_set_workspace(sg_plan_t p, void *dev_ptr, size_t bytes);

/* Defined by: the integrand parameters of the BASELINE configs / Genz families (PAPER.md:619 Test 8
 * kinds; BASELINE.json configs); f only, the quadrature Q_d^q is unchanged.
 * Replace the integrand parameters (same kind and d) by an async copy from `f` on stream s.
 * f->c / f->w may be host memory (pinned for true asynchrony) or device memory. */
int sg_update_integrand(sg_plan_t p, sg_stream_t s, const sg_integrand_desc *f);

/* Defined by: Q_d^q(f) = Eq 2.6 with Eq 2.7, evaluated by the multilevel dimension
 * iteration of PAPER.md:248-295 (Eqs 3.8-3.11, Algorithm 3.3: partial results carried one coordinate
 * at a time, "the function evaluation at any integration point is not completed until the last
 * step").
 * Enqueue the whole hot path on stream s: factor tables (K0), root pass, level-synchronous
 * frontier/leaf passes (K2/K3), deterministic reduction (K4).  out_dev (device, 2 doubles) receives
 * this plan's partial sum as a double-double (hi, lo).  Bitwise reproducible for a fixed plan.
 * Some plans (sharded fused plans, small fused plans, split frontier passes) also run one pass on
 * a plan-owned side stream: forked from s by an event recorded on s and joined back into s by an
 * event before the reduction, so the call still behaves as ordered work on s (and captures into a
 * CUDA graph on s as two branches).  Not safe to call concurrently for the same plan. */
int sg_integrate(sg_plan_t p, sg_stream_t s, double *out_dev);

/* Defined by: the outer sum of Eq 2.6 split over disjoint point sets (the shards of
 * sg_options); summation order fixed after SPEC.md:204-207 (determinism).
 * Fixed-order double-double sum of `world` gathered partials (device, 2*world doubles, rank order)
 * into result_dev (device, 2 doubles: value rounded to double, and the residual).  Writes NaN if
 * the plan's non-finite flag is set. */
int sg_finalize(sg_plan_t p, sg_stream_t s, const double *gathered_dev, int world,
                double *result_dev);

/* Defined by: Q_d^q(f), PAPER.md:65-67 (Eq 2.6), as sg_integrate + sg_finalize at world 1.
 * Synchronous convenience: H2D of nothing, runs sg_integrate + sg_finalize(world=1) on s,
 * copies the 2-double result into result_host and synchronises s. Returns SG_ENONFINITE if
 * the result is not finite. */
int sg_integrate_host(sg_plan_t p, sg_stream_t s, double *result_host);

/* Defined by: NonFiniteIntegrand.
 * Synchronously read the device status word (SG_OK or SG_ENONFINITE). */
int sg_status_word(sg_plan_t p, int *status);

/* Defined by: n_d^q = sum_{q-d+1 <= |l| <= q} n_{l_1} ... n_{l_d}.
 * Number of Smolyak points n_d^q this plan evaluates (its shard), and of the whole problem. */
int sg_plan_points(sg_plan_t p, unsigned long long *shard_points,
                   unsigned long long *total_points);

/* Defined by: DESIGN.md reading R15 (the paper does not partition work across devices).
 * Shard range actually used: [lo, hi) in depth-1 rank space, and M0 * d (= number of depth-1
 * prefixes). */
int sg_plan_range(sg_plan_t p, long long *lo, long long *hi, long long *n_depth1);

/* Defined by: the per-step partial functions f_{t-m} of PAPER.md:268-295 (Eqs 3.9-3.11): pass t
 * carries the prefixes with t active coordinates.
 * Per-pass launch statistics of the last plan: number of passes, and for pass i the number of
 * tree nodes (leaf terms) it evaluates and the frontier nodes it writes (the depth-(L-1) points that
 * k_leaf2_sym3's source tasks evaluate are counted in the last pass, whose kernel runs them).  Arrays of length >=
 * *npass (query with NULL arrays first). */
int sg_plan_passes(sg_plan_t p, int *npass, unsigned long long *terms,
                   unsigned long long *written);

/* Defined by: DESIGN.md §6 (measurement), no paper passage.
 * Host-only measurement helper: the FP64 instructions per Smolyak point of the leaf kernel variant
 * this plan runs for its dominant (last) pass — DFMA and DADD thread-instructions per point,
 * averaged over one level-2 row (midpoint, symmetric-pair and zero-tail specialisations included)
 * and, for k_leaf2_sym3, weighted with its level-3 source-task points (general oscillatory terms).
 * Used by bench.py to turn the measured kernel time into achieved FLOP/s (DFMA = 2 flops).
 * Both pointers must be non-NULL (else SG_EINVAL). */
int sg_plan_leaf_work(sg_plan_t p, double *dfma_per_point, double *dadd_per_point);

/* Defined by: the per-coordinate weights and nodes of Eq 2.7 times the
 * integrand's per-coordinate factor.
 * Debug/test hook: copy the device factor table (per level l = 2..L+1, coordinate k, node j;
 * doubles per entry: 2 real dd or 4 complex dd) and the base value to host memory. */
int sg_debug_tables(sg_plan_t p, double *table_host, size_t table_doubles, double *base_host);

/* Defined by: DESIGN.md §6 (measurement), no paper passage.
 * Profiling hook.  enable = 0 off, 1 every launch, 2 only the dominant pass (the pass with the most
 * points: two events around its launch, the other entries read 0 — bench.py's timed steps).  When enabled, sg_integrate records a CUDA event on its stream before its first
 * kernel and after each kernel.  sg_profile_read waits for the events of the LAST sg_integrate and
 * writes the device duration (ms) of each launch, in launch order:
 *   [K0 factor table, K0 base, root pass, pass 1 .. pass nfront, final reduce]
 * (the base value is computed by one extra block of the factor-table launch: its entry is ~0)
 * (SG_METHOD_COLLAPSE: [K0 factor table, K0 base, k_collapse_part, k_collapse_final]).
 * *n: in = capacity of ms[], out = number of launches (query with ms = NULL). */
int sg_profile_enable(sg_plan_t p, int enable);
int sg_profile_read(sg_plan_t p, float *ms, int *n);

/* Defined by: n_d^q and the shard partition of DESIGN.md reading R15.
 * Host-only (no device touched): the plan's counts and shard range for (d, q, rule, kind, opt).
 * Any output pointer may be NULL.  Same validation and error codes as sg_plan. */
int sg_plan_query(int d, int q, sg_rule rule, sg_kind kind, const sg_options *opt,
                  unsigned long long *shard_points, unsigned long long *total_points,
                  long long *range_lo, long long *range_hi, int *n_passes);

/* Defined by: the bijection k -> (x_{j_1}^{l_1}, ..., x_{j_d}^{l_d}) of PAPER.md:77-79 between the
 * n_d^q points and their multi-index / node tuples, with the Eq 2.6 coefficient.
 * Host-only K1 unranker (north-star subsystem 1): the `index`-th Smolyak point of the shard
 * described by (d, q, rule, kind, opt) in canonical order — the root (all-midpoint point) if the
 * shard includes it and its coefficient is nonzero, then the depth-1 subtrees r1 = lo .. hi-1, each
 * in preorder with children ordered by (k', l', j').  Outputs (host arrays of >= L entries): *t =
 * number of active coordinates; k[m], l[m] >= 2, j[m] (0-based node index of level l[m]) for
 * m < *t, ascending k; *coef = the point's Eq 2.6 coefficient (or 1 in the delta form).
 * index >= shard points -> SG_EINVAL. */
int sg_unrank(int d, int q, sg_rule rule, sg_kind kind, const sg_options *opt,
              unsigned long long index, int *t, int *k, int *l, int *j, double *coef);

/* Defined by: PAPER.md:77-79 (point bijection) and Eq 2.7's summand w_{j_1}^{l_1}...w_{j_d}^{l_d}
 * f(x) times the Eq 2.6 coefficient.
 * Device K1 + per-point evaluation (validation path): for each of the n flat
 * indices in index_dev (device, shard order of sg_unrank), enqueue on stream s the unranking and the
 * point's term evaluated on its own — coefficient * Re(B * prod of its per-coordinate factors), in
 * double-double, straight from the factor table (independent of the tree's partial products).
 * Outputs (device): points_dev[n * (1 + 3L)] = t, then (k, l, j) for m < L (-1 past depth t);
 * terms_dev[2n] = (hi, lo).  Indices outside the shard give t = -1 and a NaN term.  Builds device
 * copies of the counting tables on first use (plan-owned).  Tree method with factor arithmetic only
 * (else SG_EUNSUPPORTED). */
int sg_eval_points(sg_plan_t p, sg_stream_t s, const unsigned long long *index_dev, long long n,
                   int *points_dev, double *terms_dev);

/* Defined by: PAPER.md:103-147 (Eqs 2.10-2.13: trapezoidal, Clenshaw-Curtis, Gauss-Patterson,
 * Gauss-Legendre), mapped to [0,1] (reading R2).
 * Host-only: the library's 1-D rule of `level` on [0,1] (n_l doubles each, ascending nodes),
 * rounded once from __float128 evaluations of Eq 2.11 / Eq 2.13.  Returns n_l, or a negative
 * status (SG_EINVAL bad rule/level, SG_EUNSUPPORTED above the table limits).  x, w: host arrays of
 * at least n_l doubles. */
int sg_rule_table(sg_rule rule, int level, double *x, double *w);

/* Defined by: the ownership contract of SURVEY.md §8b.
 * Free plan-owned device memory.  The stream the plan was used on must be idle. */
int sg_destroy(sg_plan_t p);

/* Static string for a status code. */
const char *sg_strerror(int code);

#ifdef __cplusplus
}
#endif
#endif /* SG_B200_H */
