/*
 * ORACLE — test infrastructure only.  Plain, slow, obviously-correct CPU evaluation of the Smolyak
 * combination formula (Eq 2.6 with the tensor rule PAPER.md:69-71 Eq 2.7) on
 * [0,1]^d in __float128 arithmetic.  Only tests/, __graft_entry__.smoke() and bench.py's
 * cpu_baseline / --impl reference legs may load this library.  It shares no code with the CUDA
 * path (paper_2210_14313_b200/): it builds its own 1-D rule tables and evaluates f directly.
 *
 * Arithmetic: every node/weight is the double nearest to the quad value of the paper's formula
 * (readings R2-R5); sums, products and the integrand are evaluated in __float128 with
 * libquadmath (expq, cosq).  Multi-indices are visited in lexicographic order of their sparse form
 * (list of (k, l_k >= 2)), the tensor points of one multi-index by an odometer with the LAST
 * active coordinate fastest; OpenMP distributes whole top-level items (k1, l1), whose
 * quad partial sums are then added in item order, so results do not depend on the thread count.
 *
 * Pins (tests/test_oracle_pins.py): Tables 5.6-5.8 of the paper; closed forms; weight sum = 1;
 * polynomial exactness; d = 1 and L = 0 special cases; odd symmetry; brute-force tensor
 * enumeration at tiny d; the 40-digit generating-function value of Eq 2.6 for product integrands.
 */
#include <math.h>
#include <omp.h>
#include <quadmath.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#include <time.h>

typedef __float128 quad;

/* Summation / integrand arithmetic.  Default: __float128 (the parity oracle).  Compiled with
 * -DSGO_FP64 (liboracle_sg_fp64.so) the SAME program sums and evaluates f in double: the plain FP64
 * oracle, a CPU speed baseline that is not parity-grade.  The 1-D rule tables are
 * generated in quad and rounded to double in both builds (identical inputs). */
#ifdef SGO_FP64
typedef double sreal;
#define SR_EXP exp
#define SR_COS cos
#define SR_POW pow
#define SR_PI M_PI
#else
typedef quad sreal;
#define SR_EXP expq
#define SR_COS cosq
#define SR_POW powq
#define SR_PI M_PIq
#endif

enum { SGO_RULE_TRAP = 1, SGO_RULE_CC = 2, SGO_RULE_GP = 3, SGO_RULE_GL = 4 };
enum { SGO_EXP = 0, SGO_OSC = 1, SGO_PEAK = 2, SGO_GAUSS = 3, SGO_CORNER = 4, SGO_MONOMIAL = 9 };
#define SGO_MAX_LEVEL 20
#define SGO_MAX_GL 64

/* ---------------------------------------------------------------------------------------------
 * 1-D rules on [0,1]
 * ------------------------------------------------------------------------------------------- */

/* Gauss-Patterson, delayed (q = 1..10 -> N = 1, 3, 3, 7, 7, 7, 15, 15, 15, 15): level l
 * uses the Patterson rule with i extensions (2^{i+1} - 1 points) whose polynomial degree of
 * exactness, 1 for i = 0 and 3 * 2^i - 1 for i >= 1, is the first to reach that of the l-point
 * Gauss-Legendre rule, 2l - 1 (reading R16). */
static int gp_extensions(int l) {
    int i = 0;
    for (;;) {
        int exact = i == 0 ? 1 : 3 * (1 << i) - 1;
        if (exact >= 2 * l - 1) return i;
        ++i;
    }
}

/* n_l: trapezoidal and CC n_1 = 1, n_l = 2^{l-1} + 1 (Eqs 2.10, 2.11);
 * Gauss-Patterson 2^{i+1} - 1 (above); GL n_l = l. */
int sgo_node_count(int rule, int l) {
    if (l < 1) return -1;
    if (rule == SGO_RULE_CC || rule == SGO_RULE_TRAP) return l == 1 ? 1 : (1 << (l - 1)) + 1;
    if (rule == SGO_RULE_GP) return (2 << gp_extensions(l)) - 1;
    if (rule == SGO_RULE_GL) return l;
    return -1;
}

/* Clenshaw-Curtis (Eq 2.11) mapped from [-1,1] to [0,1] by x' = (x+1)/2,
 * w' = w/2 (reading R2).  Level 1 is the midpoint with weight 1 (reading R3).
 *   x_j = -cos(pi (j-1)/(n-1)),   w_1 = w_n = 1/(n(n-2)),
 *   w_j = 2/(n-1) * (1 + 2 sum'_{k=1}^{(n-1)/2} cos(2 pi (j-1) k/(n-1)) / (1 - 4k^2)),
 * sum' = last term halved.  Evaluated in quad and rounded once to double. */
static void cc_rule(int n, double *x, double *w) {
    if (n == 1) { x[0] = 0.5; w[0] = 1.0; return; }
    const quad pi = M_PIq;
    const int m = n - 1;
    for (int j = 1; j <= n; ++j) {
        quad xj = -cosq(pi * (quad)(j - 1) / (quad)m);
        x[j - 1] = (double)((xj + 1) / 2);
        quad wj;
        if (j == 1 || j == n) {
            wj = (quad)1 / ((quad)n * (quad)(n - 2));
        } else {
            quad s = 0;
            for (int k = 1; k <= m / 2; ++k) {
                quad term = cosq(2 * pi * (quad)(j - 1) * (quad)k / (quad)m) / (quad)(1 - 4 * k * k);
                if (k == m / 2) term /= 2;
                s += term;
            }
            wj = (quad)2 / (quad)m * (1 + 2 * s);
        }
        w[j - 1] = (double)(wj / 2);
    }
}

/* Legendre P_n and P_n' at t by the three-term recurrence, in quad. */
static void legendre(int n, quad t, quad *p, quad *dp) {
    quad p0 = 1, p1 = t;
    if (n == 0) { *p = 1; *dp = 0; return; }
    for (int k = 2; k <= n; ++k) {
        quad p2 = ((2 * k - 1) * t * p1 - (k - 1) * p0) / k;
        p0 = p1; p1 = p2;
    }
    *p = p1;
    *dp = n * (t * p1 - p0) / (t * t - 1);
}

/* Gauss-Legendre (Eq 2.13): zeros of P_n, weights 2/((1-t^2) P_n'(t)^2),
 * by Newton's method in quad; mapped to [0,1] (reading R2), ascending nodes. */
static void gl_rule(int n, double *x, double *w) {
    if (n == 1) { x[0] = 0.5; w[0] = 1.0; return; }
    for (int i = 1; i <= n; ++i) {
        quad t = cosq(M_PIq * ((quad)i - 0.25Q) / ((quad)n + 0.5Q));
        quad p, dp;
        for (int it = 0; it < 200; ++it) {
            legendre(n, t, &p, &dp);
            quad dt = p / dp;
            t -= dt;
            if (fabsq(dt) < 1e-33Q) break;
        }
        legendre(n, t, &p, &dp);
        quad wt = 2 / ((1 - t * t) * dp * dp);
        /* t_i descends with i; store ascending */
        x[n - i] = (double)((1 + t) / 2);
        w[n - i] = (double)(wt / 2);
    }
}

/* Trapezoidal rule (Eq 2.10): x_j = (j-1) 2^{2-l} - 1, w_j = 2^{2-l} with the first
 * and last halved, on [-1,1]; mapped to [0,1] (reading R2).  Level 1: midpoint, weight 1 (R3). */
static void trap_rule(int l, double *x, double *w) {
    if (l == 1) { x[0] = 0.5; w[0] = 1.0; return; }
    const int n = (1 << (l - 1)) + 1;
    const double h = ldexp(1.0, 2 - l);
    for (int j = 1; j <= n; ++j) {
        double xj = (j - 1) * h - 1.0, wj = h;
        if (j == 1 || j == n) wj /= 2;
        x[j - 1] = (xj + 1.0) / 2;
        w[j - 1] = wj / 2;
    }
}

/* Gauss-Legendre nodes/weights in quad on [-1,1] (descending), for the integrals below. */
static void gl_quad_rule(int n, quad *t, quad *wt) {
    for (int i = 1; i <= n; ++i) {
        quad r = cosq(M_PIq * ((quad)i - 0.25Q) / ((quad)n + 0.5Q)), p, dp;
        for (int it = 0; it < 200; ++it) {
            legendre(n, r, &p, &dp);
            quad dr = p / dp;
            r -= dr;
            if (fabsq(dr) < 1e-33Q) break;
        }
        legendre(n, r, &p, &dp);
        t[i - 1] = r;
        wt[i - 1] = 2 / ((1 - r * r) * dp * dp);
    }
}

/* sum_k a[k] P_k(x), k = 0..deg, by Clenshaw's recurrence (P_{k+1} = ((2k+1) x P_k - k P_{k-1})/(k+1)). */
static quad legendre_series(const quad *a, int deg, quad x) {
    quad b1 = 0, b2 = 0;
    for (int k = deg; k >= 1; --k) {
        /* alpha_k(x) = (2k+1) x / (k+1), beta_{k+1} = -(k+1)/(k+2) */
        quad b0 = a[k] + (2 * k + 1) * x / (k + 1) * b1 - (quad)(k + 1) / (k + 2) * b2;
        b2 = b1; b1 = b0;
    }
    return a[0] + x * b1 - 0.5Q * b2;
}

/* Solve A z = b (n x n, row-major, destroyed) by Gaussian elimination with partial pivoting. */
static int solve_quad(int n, quad *A, quad *b, quad *z) {
    for (int c = 0; c < n; ++c) {
        int piv = c;
        for (int r = c + 1; r < n; ++r) if (fabsq(A[r * n + c]) > fabsq(A[piv * n + c])) piv = r;
        if (A[piv * n + c] == 0) return -1;
        if (piv != c) {
            for (int j = 0; j < n; ++j) { quad t = A[c * n + j]; A[c * n + j] = A[piv * n + j]; A[piv * n + j] = t; }
            quad t = b[c]; b[c] = b[piv]; b[piv] = t;
        }
        for (int r = c + 1; r < n; ++r) {
            quad f = A[r * n + c] / A[c * n + c];
            for (int j = c; j < n; ++j) A[r * n + j] -= f * A[c * n + j];
            b[r] -= f * b[c];
        }
    }
    for (int c = n - 1; c >= 0; --c) {
        quad v = b[c];
        for (int j = c + 1; j < n; ++j) v -= A[c * n + j] * z[j];
        z[c] = v / A[c * n + c];
    }
    return 0;
}

/* Gauss-Patterson rule with `ext` extensions (Eq 2.12), on [0,1], written from the
 * definition with n = 1: the nodes are the zero of P_1 and the zeros of G_1, ..., G_ext, where G_i has
 * degree 2^{i-1}(n+1) = 2^i and is orthogonal to every polynomial of degree < 2^i with respect to the
 * weight P_1(x) G_1(x) ... G_{i-1}(x) on [-1,1].  Each G_i is monic-in-P (G_i = P_{2^i} + sum a_k P_k),
 * stored by its Legendre coefficients.  G_i is even and the weight odd, so the orthogonality
 * conditions against even P_k hold identically; the conditions against odd P_k (k < 2^i) determine
 * the even coefficients a_k (k < 2^i).  Zeros: sign changes of G_i on a fine grid in arccos space,
 * refined by bisection.  Weights: the rule is interpolatory, so w solves the moment equations
 * sum_j w_j P_k(x_j) = 2 delta_{k0}, k = 0 .. N-1.  All in quad, rounded once to double. */
#define GP_MAXN 63
static int gp_rule(int ext, double *x, double *w) {
    static quad G[7][GP_MAXN + 2];          /* Legendre coefficients of G_1 .. G_ext */
    quad nodes[GP_MAXN];
    int N = 1;
    nodes[0] = 0;                             /* zero of P_1 */
    for (int i = 1; i <= ext; ++i) {
        const int deg = 1 << i, nu = deg / 2;
        const int nq = (3 * deg) / 2 + 2;     /* Gauss points: exact for the integrand degree < 2 nq */
        quad *gt = malloc(sizeof(quad) * nq), *gw = malloc(sizeof(quad) * nq);
        quad *A = calloc((size_t)nu * nu, sizeof(quad)), *b = calloc(nu, sizeof(quad));
        quad *z = calloc(nu, sizeof(quad));
        gl_quad_rule(nq, gt, gw);
        for (int q = 0; q < nq; ++q) {
            quad wgt = gt[q];                 /* P_1 */
            for (int j = 1; j < i; ++j) wgt *= legendre_series(G[j], 1 << j, gt[q]);
            for (int r = 0; r < nu; ++r) {
                quad pk, dpk, pc, dpc, ptop, dtop;
                legendre(2 * r + 1, gt[q], &pk, &dpk);
                legendre(deg, gt[q], &ptop, &dtop);
                for (int c = 0; c < nu; ++c) {
                    legendre(2 * c, gt[q], &pc, &dpc);
                    A[r * nu + c] += gw[q] * wgt * pk * pc;
                }
                b[r] -= gw[q] * wgt * pk * ptop;
            }
        }
        if (solve_quad(nu, A, b, z)) return -1;
        for (int k = 0; k <= deg; ++k) G[i][k] = 0;
        G[i][deg] = 1;
        for (int c = 0; c < nu; ++c) G[i][2 * c] = z[c];
        free(gt); free(gw); free(A); free(b); free(z);
        /* zeros of G_i */
        const int grid = 1 << 14;
        int found = 0;
        quad xa = -1, fa = legendre_series(G[i], deg, xa);
        for (int g = 1; g <= grid; ++g) {
            quad xb = -cosq(M_PIq * g / grid), fb = legendre_series(G[i], deg, xb);
            if (g == grid) xb = 1;
            if ((fa < 0) != (fb < 0)) {
                quad lo = xa, hi = xb, flo = fa;
                for (int it = 0; it < 300 && hi - lo > 1e-36Q; ++it) {
                    quad mid = (lo + hi) / 2, fm = legendre_series(G[i], deg, mid);
                    if ((fm < 0) == (flo < 0)) { lo = mid; flo = fm; } else hi = mid;
                }
                if (N + found >= GP_MAXN) return -1;
                nodes[N + found++] = (lo + hi) / 2;
            }
            xa = xb; fa = fb;
        }
        if (found != deg) return -1;
        N += found;
    }
    /* ascending order */
    for (int a = 1; a < N; ++a)
        for (int c = a; c > 0 && nodes[c] < nodes[c - 1]; --c) { quad t = nodes[c]; nodes[c] = nodes[c - 1]; nodes[c - 1] = t; }
    quad *A = calloc((size_t)N * N, sizeof(quad)), *b = calloc(N, sizeof(quad)), *z = calloc(N, sizeof(quad));
    for (int k = 0; k < N; ++k) {
        for (int j = 0; j < N; ++j) {
            quad p, dp;
            legendre(k, nodes[j], &p, &dp);
            A[k * N + j] = p;
        }
        b[k] = k == 0 ? 2 : 0;
    }
    int rc = solve_quad(N, A, b, z);
    for (int j = 0; j < N && !rc; ++j) {
        x[j] = (double)((1 + nodes[j]) / 2);
        w[j] = (double)(z[j] / 2);
    }
    free(A); free(b); free(z);
    return rc ? -1 : N;
}

/* Public: fill nodes/weights of level l, return n_l (or -1). */
int sgo_rule(int rule, int l, double *x, double *w) {
    int n = sgo_node_count(rule, l);
    if (n < 0) return -1;
    if (rule == SGO_RULE_CC) {
        if (l > SGO_MAX_LEVEL) return -1;
        cc_rule(n, x, w);
    } else if (rule == SGO_RULE_TRAP) {
        if (l > SGO_MAX_LEVEL) return -1;
        trap_rule(l, x, w);
    } else if (rule == SGO_RULE_GP) {
        if (n > GP_MAXN) return -1;
        if (gp_rule(gp_extensions(l), x, w) != n) return -1;
    } else {
        if (n > SGO_MAX_GL) return -1;
        gl_rule(n, x, w);
    }
    return n;
}

/* ---------------------------------------------------------------------------------------------
 * Integrand (BASELINE.json configs; PAPER.md:619 Test 8 kinds), evaluated at a full point x.
 * ------------------------------------------------------------------------------------------- */
typedef struct {
    int d, kind;
    const double *c, *w;
    double u;
    sreal two_pi_u;     /* 2 pi u */
    sreal *cinv2;       /* c_k^-2 (peak) */
    sreal s_mid;        /* sum_k c_k / 2 (exp/osc) or sum_k c_k^2 (1/2 - w_k)^2 (gauss) */
    sreal peak_mid;     /* prod_k 1/(c_k^-2 + (1/2 - w_k)^2) */
} integrand;

/* Plain O(d) evaluation: f(x_1..x_d) exactly as written in BASELINE.json. */
static sreal f_plain(const integrand *F, const double *x) {
    const int d = F->d;
    sreal s = 0, p = 1;
    switch (F->kind) {
    case SGO_EXP:
        for (int k = 0; k < d; ++k) s += (sreal)F->c[k] * (sreal)x[k];
        return SR_EXP(s);
    case SGO_OSC:
        for (int k = 0; k < d; ++k) s += (sreal)F->c[k] * (sreal)x[k];
        return SR_COS(F->two_pi_u + s);
    case SGO_PEAK:
        for (int k = 0; k < d; ++k) {
            sreal t = (sreal)x[k] - (sreal)F->w[k];
            p *= 1 / (F->cinv2[k] + t * t);
        }
        return p;
    case SGO_GAUSS:
        for (int k = 0; k < d; ++k) {
            sreal t = (sreal)x[k] - (sreal)F->w[k];
            s += (sreal)F->c[k] * (sreal)F->c[k] * t * t;
        }
        return SR_EXP(-s);
    case SGO_CORNER: /* Genz corner peak: (1 + sum_k c_k x_k)^-(d+1) */
        for (int k = 0; k < d; ++k) s += (sreal)F->c[k] * (sreal)x[k];
        return SR_POW(1 + s, -(sreal)(d + 1));
    case SGO_MONOMIAL: /* test-only: prod x_k^{alpha_k}, alpha_k = (int) w[k] */
        for (int k = 0; k < d; ++k) {
            int a = (int)F->w[k];
            for (int e = 0; e < a; ++e) p *= (sreal)x[k];
        }
        return p;
    }
    return (sreal)NAN;
}

/* "Active" evaluation: the same f, using that every inactive coordinate sits at the midpoint 1/2
 * (level 1, reading R3), so sum_k c_k x_k = sum_k c_k/2 + sum_active c_k (x_k - 1/2) exactly in
 * real arithmetic (and the analogues for gauss/peak).  O(#active) per point; cross-checked
 * against f_plain in tests. */
static sreal f_active(const integrand *F, int t, const int *ak, const double *ax) {
    sreal s = 0, p;
    switch (F->kind) {
    case SGO_EXP:
        for (int m = 0; m < t; ++m) s += (sreal)F->c[ak[m]] * ((sreal)ax[m] - (sreal)0.5);
        return SR_EXP(F->s_mid + s);
    case SGO_OSC:
        for (int m = 0; m < t; ++m) s += (sreal)F->c[ak[m]] * ((sreal)ax[m] - (sreal)0.5);
        return SR_COS(F->two_pi_u + F->s_mid + s);
    case SGO_CORNER:
        for (int m = 0; m < t; ++m) s += (sreal)F->c[ak[m]] * ((sreal)ax[m] - (sreal)0.5);
        return SR_POW(1 + F->s_mid + s, -(sreal)(F->d + 1));
    case SGO_GAUSS:
        for (int m = 0; m < t; ++m) {
            int k = ak[m];
            sreal c2 = (sreal)F->c[k] * (sreal)F->c[k];
            sreal a = (sreal)ax[m] - (sreal)F->w[k], b = (sreal)0.5 - (sreal)F->w[k];
            s += c2 * (a * a - b * b);
        }
        return SR_EXP(-(F->s_mid + s));
    case SGO_PEAK:
        p = F->peak_mid;
        for (int m = 0; m < t; ++m) {
            int k = ak[m];
            sreal a = (sreal)ax[m] - (sreal)F->w[k], b = (sreal)0.5 - (sreal)F->w[k];
            p *= (F->cinv2[k] + b * b) / (F->cinv2[k] + a * a);
        }
        return p;
    }
    return (sreal)NAN;
}

/* ---------------------------------------------------------------------------------------------
 * Combination formula, Eq 2.6 with q = d + L:  |l| = d + e, e in [max(0, L-d+1), L],
 * coefficient (-1)^{q-|l|} C(d-1, q-|l|) = (-1)^{L-e} C(d-1, L-e).
 * ------------------------------------------------------------------------------------------- */
static quad binom_q(int n, int k) {
    if (k < 0 || k > n) return 0;
    quad r = 1;
    for (int i = 1; i <= k; ++i) r = r * (quad)(n - k + i) / (quad)i;
    return rintq(r);
}

typedef struct {
    int d, L, rule, eval_mode, emin;
    const integrand *F;
    int nl[SGO_MAX_LEVEL + 2];
    double *X[SGO_MAX_LEVEL + 2], *W[SGO_MAX_LEVEL + 2];
    sreal coef[SGO_MAX_LEVEL + 2];
    int64_t M0;                      /* number of depth-1 (k1,l1,j1) triples per coordinate */
    int64_t lo, hi;                  /* shard: depth-1 lexicographic range [lo, hi) */
    int64_t stride;                  /* sample: every stride-th depth-2 subtree of each top-level item */
    int count_only;                  /* count the selected points, evaluate nothing */
} problem;

typedef struct {
    int t;                           /* number of active coordinates */
    int ak[SGO_MAX_LEVEL + 2], al[SGO_MAX_LEVEL + 2];
    double *xfull;                   /* full point for the plain evaluator */
    sreal sum;
    int64_t npoints;
} walker;

/* Lexicographic rank of a depth-1 triple (k1, l1, j1): k1 * M0 + sum_{l<l1} n_l + j1. */
static int64_t depth1_rank(const problem *P, int k1, int l1, int j1) {
    int64_t r = (int64_t)k1 * P->M0;
    for (int l = 2; l < l1; ++l) r += P->nl[l];
    return r + j1;
}

/* Tensor rule of one multi-index (Eq 2.7): odometer over the nodes of the active coordinates. */
static void tensor_sum(const problem *P, walker *Wk, int e) {
    const int t = Wk->t;
    int j[SGO_MAX_LEVEL + 2];
    double ax[SGO_MAX_LEVEL + 2];
    int jlo0 = 0, jhi0 = t > 0 ? P->nl[Wk->al[0]] : 1;
    if (t > 0) {   /* shard restriction on the first active coordinate's node */
        int64_t base = depth1_rank(P, Wk->ak[0], Wk->al[0], 0);
        int64_t a = P->lo - base, b = P->hi - base;
        if (a > jlo0) jlo0 = (int)(a < jhi0 ? a : jhi0);
        if (b < jhi0) jhi0 = (int)(b > jlo0 ? b : jlo0);
        if (jlo0 >= jhi0) return;
    }
    if (P->count_only) {
        int64_t n = t > 0 ? jhi0 - jlo0 : 1;
        for (int m = 1; m < t; ++m) n *= P->nl[Wk->al[m]];
        Wk->npoints += n;
        return;
    }
    for (int m = 0; m < t; ++m) j[m] = 0;
    if (t > 0) j[0] = jlo0;
    sreal acc = 0;
    for (;;) {
        sreal wprod = 1;
        for (int m = 0; m < t; ++m) {
            wprod *= (sreal)P->W[Wk->al[m]][j[m]];
            ax[m] = P->X[Wk->al[m]][j[m]];
        }
        sreal fx;
        if (P->eval_mode == 0) {
            for (int m = 0; m < t; ++m) Wk->xfull[Wk->ak[m]] = ax[m];
            fx = f_plain(P->F, Wk->xfull);
        } else {
            fx = f_active(P->F, t, Wk->ak, ax);
        }
        acc += wprod * fx;
        Wk->npoints++;
        /* advance odometer, last active coordinate fastest */
        int m = t - 1;
        while (m >= 0) {
            int lim = (m == 0) ? jhi0 : P->nl[Wk->al[m]];
            if (++j[m] < lim) break;
            j[m] = (m == 0) ? jlo0 : 0;
            --m;
        }
        if (m < 0) break;
    }
    if (P->eval_mode == 0)
        for (int m = 0; m < t; ++m) Wk->xfull[Wk->ak[m]] = 0.5;
    Wk->sum += P->coef[e] * acc;
}

/* Depth-first walk over sparse multi-indices in lexicographic order. */
static void walk(const problem *P, walker *Wk, int kstart, int e) {
    if (e >= P->emin) tensor_sum(P, Wk, e);
    for (int k = kstart; k < P->d; ++k) {
        for (int l = 2; l <= P->L + 1 - e; ++l) {
            Wk->ak[Wk->t] = k; Wk->al[Wk->t] = l; Wk->t++;
            walk(P, Wk, k + 1, e + l - 1);
            Wk->t--;
        }
    }
}

/*
 * sgo_integrate: A(q = d + L, d) f on [0,1]^d, restricted to the points whose first active
 * coordinate triple (k1, l1, j1) has depth-1 lexicographic rank in [lo, hi), plus the all-midpoint
 * point when include_root != 0 (lo = 0, hi = -1 means "everything").
 * eval_mode: 0 = plain O(d) integrand, 1 = active-coordinate identity (see f_active).
 * Outputs: out_hilo[0] + out_hilo[1] = quad result rounded to a double pair; out_str = "%.36Qe";
 * out_npoints = tensor points evaluated; out_seconds = wall time of the summation.
 * Returns 0, or -1 on bad arguments.
 * sgo_integrate_ex adds: stride (> 1: only the points of every stride-th depth-2 multi-index subtree
 * (k1, l1, k2, l2, ...) of each top-level item (k1, l1), in walk order, the counter starting at the
 * item's index: an evenly spread sample of the whole tree for CPU timing; the root and the depth-1
 * multi-indices are not sampled) and count_only (return the number of selected points in
 * out_npoints, evaluate nothing).
 */
int sgo_integrate_ex(int d, int L, int rule, int kind, const double *c, const double *w, double u,
                     long long lo, long long hi, long long stride, int include_root, int eval_mode,
                     int nthreads, int count_only, double *out_hilo, char *out_str,
                     long long *out_npoints, double *out_seconds) {
    if (stride < 1) return -1;
    if (d < 1 || L < 0 || L + 1 > SGO_MAX_LEVEL || !c) return -1;
    if ((kind == SGO_PEAK || kind == SGO_GAUSS || kind == SGO_MONOMIAL) && !w) return -1;
    if (kind == SGO_MONOMIAL && eval_mode != 0) return -1;
    if (kind == SGO_CORNER) {   /* 1 + sum c_k x_k > 0 on the cube */
        double m = 1.0;
        for (int k = 0; k < d; ++k) m += c[k] < 0 ? c[k] : 0.0;
        if (!(m > 0)) return -1;
    }
    problem P;
    memset(&P, 0, sizeof P);
    P.d = d; P.L = L; P.rule = rule; P.eval_mode = eval_mode;
    P.emin = L - d + 1 > 0 ? L - d + 1 : 0;
    for (int l = 1; l <= L + 1; ++l) {
        int n = sgo_node_count(rule, l);
        if (n < 0 || (rule == SGO_RULE_GL && n > SGO_MAX_GL)) return -1;
        P.nl[l] = n;
        P.X[l] = (double *)malloc(sizeof(double) * n);
        P.W[l] = (double *)malloc(sizeof(double) * n);
        sgo_rule(rule, l, P.X[l], P.W[l]);
    }
    for (int e = 0; e <= L; ++e) {
        quad b = binom_q(d - 1, L - e);
        P.coef[e] = (sreal)((L - e) % 2 ? -b : b);   /* exact in double too: |C| < 2^53 (plan limits) */
    }
    P.M0 = 0;
    for (int l = 2; l <= L + 1; ++l) P.M0 += P.nl[l];
    P.lo = lo; P.hi = hi < 0 ? (int64_t)d * P.M0 + 1 : hi;
    P.stride = stride; P.count_only = count_only;

    integrand F;
    memset(&F, 0, sizeof F);
    F.d = d; F.kind = kind; F.c = c; F.w = w; F.u = u;
    F.two_pi_u = 2 * SR_PI * (sreal)u;
    F.cinv2 = (sreal *)malloc(sizeof(sreal) * d);
    F.s_mid = 0; F.peak_mid = 1;
    for (int k = 0; k < d; ++k) {
        F.cinv2[k] = 1 / ((sreal)c[k] * (sreal)c[k]);
        if (kind == SGO_EXP || kind == SGO_OSC || kind == SGO_CORNER) F.s_mid += (sreal)c[k] / 2;
        if (kind == SGO_GAUSS) {
            sreal b = (sreal)0.5 - (sreal)w[k];
            F.s_mid += (sreal)c[k] * (sreal)c[k] * b * b;
        }
        if (kind == SGO_PEAK) {
            sreal b = (sreal)0.5 - (sreal)w[k];
            F.peak_mid *= 1 / (F.cinv2[k] + b * b);
        }
    }
    P.F = &F;

    if (stride > 1) {
        /* Timing sample: the depth-2 multi-index subtrees (k1, l1, k2, l2) in lexicographic order,
         * numbered 0, 1, 2, ...; every stride-th one, starting at stride / 2; OpenMP over the
         * selected subtrees, partial sums added in list order.  The root and the depth-1
         * multi-indices are not part of the sample. */
        int64_t nsel = 0, cap = 1024, cnt = 0;
        int *U = (int *)malloc(sizeof(int) * 4 * cap);
        for (int k1 = 0; k1 < d; ++k1)
            for (int l1 = 2; l1 <= L + 1; ++l1) {
                for (int k2 = k1 + 1; k2 < d; ++k2)
                    for (int l2 = 2; l2 <= L + 1 - (l1 - 1); ++l2, ++cnt) {
                        if (cnt % stride != stride / 2) continue;
                        if (nsel == cap) { cap *= 2; U = (int *)realloc(U, sizeof(int) * 4 * cap); }
                        U[4 * nsel] = k1; U[4 * nsel + 1] = l1; U[4 * nsel + 2] = k2; U[4 * nsel + 3] = l2;
                        ++nsel;
                    }
            }
        sreal *usum = (sreal *)calloc(nsel > 0 ? nsel : 1, sizeof(sreal));
        int64_t *upts = (int64_t *)calloc(nsel > 0 ? nsel : 1, sizeof(int64_t));
        if (nthreads > 0) omp_set_num_threads(nthreads);
        struct timespec s0, s1;
        clock_gettime(CLOCK_MONOTONIC, &s0);
#pragma omp parallel
        {
            walker Wk;
            memset(&Wk, 0, sizeof Wk);
            Wk.xfull = (double *)malloc(sizeof(double) * d);
            for (int k = 0; k < d; ++k) Wk.xfull[k] = 0.5;
#pragma omp for schedule(dynamic, 1)
            for (int64_t i = 0; i < nsel; ++i) {
                Wk.sum = 0; Wk.npoints = 0; Wk.t = 2;
                Wk.ak[0] = U[4 * i]; Wk.al[0] = U[4 * i + 1]; Wk.ak[1] = U[4 * i + 2]; Wk.al[1] = U[4 * i + 3];
                walk(&P, &Wk, Wk.ak[1] + 1, Wk.al[0] - 1 + Wk.al[1] - 1);
                usum[i] = Wk.sum; upts[i] = Wk.npoints;
            }
            free(Wk.xfull);
        }
        sreal tot = 0;
        int64_t np = 0;
        for (int64_t i = 0; i < nsel; ++i) { tot += usum[i]; np += upts[i]; }
        clock_gettime(CLOCK_MONOTONIC, &s1);
        double hd = (double)tot;
        if (out_hilo) { out_hilo[0] = hd; out_hilo[1] = (double)(tot - (sreal)hd); }
        if (out_str) quadmath_snprintf(out_str, 64, "%.36Qe", (quad)tot);
        if (out_npoints) *out_npoints = np;
        if (out_seconds) *out_seconds = (s1.tv_sec - s0.tv_sec) + 1e-9 * (s1.tv_nsec - s0.tv_nsec);
        for (int l = 1; l <= L + 1; ++l) { free(P.X[l]); free(P.W[l]); }
        free(F.cinv2); free(U); free(usum); free(upts);
        return 0;
    }

    /* top-level items: (k1, l1) for k1 in [0,d), l1 in [2, L+1]; item sums added in order */
    const int nitems = d * L;
    sreal *item_sum = (sreal *)calloc(nitems > 0 ? nitems : 1, sizeof(sreal));
    int64_t *item_pts = (int64_t *)calloc(nitems > 0 ? nitems : 1, sizeof(int64_t));
    if (nthreads > 0) omp_set_num_threads(nthreads);
    struct timespec t0, t1;
    clock_gettime(CLOCK_MONOTONIC, &t0);

    sreal root_sum = 0;
    int64_t root_pts = 0;
    if (include_root && P.emin == 0) {
        walker Wk;
        memset(&Wk, 0, sizeof Wk);
        Wk.xfull = (double *)malloc(sizeof(double) * d);
        for (int k = 0; k < d; ++k) Wk.xfull[k] = 0.5;
        tensor_sum(&P, &Wk, 0);
        root_sum = Wk.sum; root_pts = Wk.npoints;
        free(Wk.xfull);
    }

#pragma omp parallel
    {
        walker Wk;
        memset(&Wk, 0, sizeof Wk);
        Wk.xfull = (double *)malloc(sizeof(double) * d);
        for (int k = 0; k < d; ++k) Wk.xfull[k] = 0.5;
#pragma omp for schedule(dynamic, 1)
        for (int it = 0; it < nitems; ++it) {
            int k1 = it / L, l1 = 2 + it % L;
            int64_t r0 = depth1_rank(&P, k1, l1, 0), r1 = r0 + P.nl[l1];
            if (r1 <= P.lo || r0 >= P.hi) continue;
            Wk.sum = 0; Wk.npoints = 0; Wk.t = 1;
            Wk.ak[0] = k1; Wk.al[0] = l1;
            walk(&P, &Wk, k1 + 1, l1 - 1);
            item_sum[it] = Wk.sum; item_pts[it] = Wk.npoints;
        }
        free(Wk.xfull);
    }
    sreal total = root_sum;
    int64_t npts = root_pts;
    for (int it = 0; it < nitems; ++it) { total += item_sum[it]; npts += item_pts[it]; }
    clock_gettime(CLOCK_MONOTONIC, &t1);

    double hi_d = (double)total;
    double lo_d = (double)(total - (sreal)hi_d);
    if (out_hilo) { out_hilo[0] = hi_d; out_hilo[1] = lo_d; }
    if (out_str) quadmath_snprintf(out_str, 64, "%.36Qe", (quad)total);
    if (out_npoints) *out_npoints = npts;
    if (out_seconds) *out_seconds = (t1.tv_sec - t0.tv_sec) + 1e-9 * (t1.tv_nsec - t0.tv_nsec);
    for (int l = 1; l <= L + 1; ++l) { free(P.X[l]); free(P.W[l]); }
    free(F.cinv2); free(item_sum); free(item_pts);
    return 0;
}

int sgo_integrate(int d, int L, int rule, int kind, const double *c, const double *w, double u,
                  long long lo, long long hi, int include_root, int eval_mode, int nthreads,
                  double *out_hilo, char *out_str, long long *out_npoints, double *out_seconds) {
    return sgo_integrate_ex(d, L, rule, kind, c, w, u, lo, hi, 1, include_root, eval_mode, nthreads, 0,
                            out_hilo, out_str, out_npoints, out_seconds);
}

/* Single-point evaluation (test hook): f at a full point x, plain and active forms. */
int sgo_eval_point(int d, int kind, const double *c, const double *w, double u, const double *x,
                   double *out_plain, double *out_active) {
    integrand F;
    memset(&F, 0, sizeof F);
    F.d = d; F.kind = kind; F.c = c; F.w = w; F.u = u;
    F.two_pi_u = 2 * SR_PI * (sreal)u;
    F.cinv2 = (sreal *)malloc(sizeof(sreal) * d);
    F.peak_mid = 1;
    int *ak = (int *)malloc(sizeof(int) * d);
    double *ax = (double *)malloc(sizeof(double) * d);
    int t = 0;
    for (int k = 0; k < d; ++k) {
        F.cinv2[k] = 1 / ((sreal)c[k] * (sreal)c[k]);
        if (kind == SGO_EXP || kind == SGO_OSC || kind == SGO_CORNER) F.s_mid += (sreal)c[k] / 2;
        if (kind == SGO_GAUSS) { sreal b = (sreal)0.5 - (sreal)w[k]; F.s_mid += (sreal)c[k] * (sreal)c[k] * b * b; }
        if (kind == SGO_PEAK) { sreal b = (sreal)0.5 - (sreal)w[k]; F.peak_mid *= 1 / (F.cinv2[k] + b * b); }
        if (x[k] != 0.5) { ak[t] = k; ax[t] = x[k]; ++t; }
    }
    sreal a = f_plain(&F, x);
    sreal b = kind == SGO_MONOMIAL ? a : f_active(&F, t, ak, ax);
    out_plain[0] = (double)a; out_plain[1] = (double)(a - (sreal)out_plain[0]);
    out_active[0] = (double)b; out_active[1] = (double)(b - (sreal)out_active[0]);
    free(F.cinv2); free(ak); free(ax);
    return 0;
}
