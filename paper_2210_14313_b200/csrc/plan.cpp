// plan.cpp — host planning for the B200 Smolyak path (compiled by g++; uses __float128).
//
// K0 (rules):  trapezoidal (Eq 2.10), Clenshaw-Curtis (Eq 2.11),
//              Gauss-Patterson (Eq 2.12; delayed sequence of PAPER.md:615) and
//              Gauss-Legendre (Eq 2.13) on [0,1] (reading R2), evaluated in
//              __float128 and rounded once to double.
// K1 (counts): per-depth segment counts of the prefix tree, subtree point counts (PAPER.md:73-75
//              n_d^q), balanced shard ranges of depth-1 subtrees, launch geometry.
#include "plan.h"

#include <quadmath.h>

#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>

#include "../../include/sg_b200.h"

typedef __float128 q128;
typedef unsigned __int128 u128;

// Gauss-Patterson level l -> Patterson rule index k (2^k - 1 points): the smallest rule whose degree
// of exactness (1 for k = 1, 3 * 2^(k-1) - 1 for k >= 2) reaches 2l - 1, the exactness of the
// l-point Gauss-Legendre rule.  Gives the "delayed" sequence n_l = 1, 3, 3, 7, 7, 7, 15, ... that
// PAPER.md:615 lists for r = 3 (reading R16), and reproduces the paper's node counts (Tables 4.1,
// 4.3, 4.5, 4.6).
static int gp_index(int l) {
    int k = 1;
    while ((k == 1 ? 1 : 3 * (1 << (k - 1)) - 1) < 2 * l - 1) ++k;
    return k;
}

int host_node_count(int rule, int l) {
    if (l < 1) return -1;
    if (rule == SG_RULE_CLENSHAW_CURTIS || rule == SG_RULE_TRAPEZOIDAL) return l == 1 ? 1 : (1 << (l - 1)) + 1;
    if (rule == SG_RULE_GAUSS_LEGENDRE) return l;
    if (rule == SG_RULE_GAUSS_PATTERSON) return (1 << gp_index(l)) - 1;
    return -1;
}

// CC on [0,1]: x_j = (1 - cos(pi (j-1)/(n-1)))/2 = sin^2(pi (j-1) / (2(n-1)));
// w_1 = w_n = 1/(2 n (n-2)); w_j = 1/(n-1) (1 + 2 sum'_{k=1}^{(n-1)/2} cos(2 pi (j-1) k/(n-1))/(1-4k^2)).
static void cc_rule_q(int n, double *x, double *w) {
    if (n == 1) {
        x[0] = 0.5;
        w[0] = 1.0;
        return;
    }
    const int m = n - 1, half = m / 2;
    for (int j = 0; j < n; ++j) {
        q128 s = sinq(M_PIq * (q128)j / (q128)(2 * m));
        x[j] = (double)(s * s);
        if (j == 0 || j == m) {
            w[j] = (double)((q128)1 / ((q128)2 * (q128)n * (q128)(n - 2)));
            continue;
        }
        q128 acc = 0;
        for (int k = half; k >= 1; --k) {   // summed from the last term (halved) down
            q128 term = cosq((q128)2 * M_PIq * (q128)j * (q128)k / (q128)m) / (q128)(1 - 4 * k * k);
            acc += (k == half) ? term / 2 : term;
        }
        w[j] = (double)(((q128)1 + 2 * acc) / (q128)m);
    }
}

// GL on [0,1]: roots of P_n by Newton from Tricomi's initial guess, weights 2/((1-t^2) P_n'(t)^2),
// mapped x = (1+t)/2, w/2.
static void gl_rule_q(int n, double *x, double *w) {
    if (n == 1) {
        x[0] = 0.5;
        w[0] = 1.0;
        return;
    }
    for (int i = 0; i < n; ++i) {
        // ascending root i: t ~ -cos(pi (4(i+1) - 1)/(4n + 2)) corrected
        q128 th = M_PIq * (q128)(4 * (i + 1) - 1) / (q128)(4 * n + 2);
        q128 t = -cosq(th) * (1 - (q128)(n - 1) / ((q128)8 * n * n * n));
        q128 p1 = 0, p0 = 0, dp = 0;
        for (int it = 0; it < 100; ++it) {
            p0 = 1;
            p1 = t;
            for (int k = 2; k <= n; ++k) {
                q128 p2 = ((q128)(2 * k - 1) * t * p1 - (q128)(k - 1) * p0) / (q128)k;
                p0 = p1;
                p1 = p2;
            }
            dp = (q128)n * (p0 - t * p1) / (1 - t * t);
            q128 step = p1 / dp;
            t -= step;
            if (fabsq(step) <= 1e-34Q * (1 + fabsq(t))) break;
        }
        p0 = 1;
        p1 = t;
        for (int k = 2; k <= n; ++k) {
            q128 p2 = ((q128)(2 * k - 1) * t * p1 - (q128)(k - 1) * p0) / (q128)k;
            p0 = p1;
            p1 = p2;
        }
        dp = (q128)n * (p0 - t * p1) / (1 - t * t);
        x[i] = (double)((1 + t) / 2);
        w[i] = (double)((q128)1 / ((1 - t * t) * dp * dp));
    }
}

// Trapezoidal rule (Eq 2.10) on [0,1]: x_j = (j-1)/(n-1), weights 1/(n-1) with the
// first and last halved (the paper's h = 2^{2-l} on [-1,1], halved by the map); level 1 = midpoint,
// weight 1 (reading R3).  All values are exact dyadic rationals.
static void trap_rule_q(int n, double *x, double *w) {
    if (n == 1) {
        x[0] = 0.5;
        w[0] = 1.0;
        return;
    }
    const int m = n - 1;
    for (int j = 0; j < n; ++j) {
        x[j] = (double)j / (double)m;
        w[j] = (j == 0 || j == m) ? 0.5 / (double)m : 1.0 / (double)m;
    }
}

// Gauss-Legendre n-point rule on [-1,1] in quad (ascending), for the Patterson construction.
static void gl_quad(int n, std::vector<q128> &t, std::vector<q128> &wt) {
    t.assign(n, 0);
    wt.assign(n, 0);
    for (int i = 0; i < n; ++i) {
        q128 th = M_PIq * (q128)(4 * (i + 1) - 1) / (q128)(4 * n + 2);
        q128 r = -cosq(th), p0 = 1, p1 = r, dp = 0;
        for (int it = 0; it < 100; ++it) {
            p0 = 1;
            p1 = r;
            for (int k = 2; k <= n; ++k) {
                q128 p2 = ((q128)(2 * k - 1) * r * p1 - (q128)(k - 1) * p0) / (q128)k;
                p0 = p1;
                p1 = p2;
            }
            dp = (q128)n * (p0 - r * p1) / (1 - r * r);
            q128 step = p1 / dp;
            r -= step;
            if (fabsq(step) <= 1e-34Q) break;
        }
        p0 = 1;
        p1 = r;
        for (int k = 2; k <= n; ++k) {
            q128 p2 = ((q128)(2 * k - 1) * r * p1 - (q128)(k - 1) * p0) / (q128)k;
            p0 = p1;
            p1 = p2;
        }
        dp = (q128)n * (p0 - r * p1) / (1 - r * r);
        t[i] = r;
        wt[i] = (q128)2 / ((1 - r * r) * dp * dp);
    }
}

// P_0(x) .. P_N(x) by the three-term recurrence
static void legendre_all(int N, q128 x, q128 *P) {
    P[0] = 1;
    if (N >= 1) P[1] = x;
    for (int k = 2; k <= N; ++k) P[k] = ((q128)(2 * k - 1) * x * P[k - 1] - (q128)(k - 1) * P[k - 2]) / (q128)k;
}

// Gauss-Patterson rule k (2^k - 1 points) on [-1,1] in quad (Eq 2.12): start from the
// 1-point Gauss rule (the zero of P_1) and extend m -> 2m + 1 points, m = 2^s - 1: the m + 1 new nodes
// are the zeros of G = P_{m+1} + sum_j a_j P_j, orthogonal to every polynomial of degree <= m with
// respect to the weight p_m(t) = prod (t - old nodes).  G has the parity of m + 1 (even), so only the
// equations against odd P_i and the even coefficients a_j remain: a square (m+1)/2 system, solved
// in quad with partial pivoting (integrals by Gauss-Legendre, exact for degree 3m + 1).  The new zeros
// interlace the old nodes: one by bisection in each gap.  Weights: interpolatory, w_j = integral of
// the Lagrange basis polynomial (Gauss-Legendre, exact).  Returns false if a bracket fails.
static bool gp_quad(int k, std::vector<q128> &t, std::vector<q128> &wt) {
    t.assign(1, (q128)0);
    for (int s = 1; s < k; ++s) {
        const int m = (int)t.size(), nu = (m + 1) / 2, nq = (3 * m + 3) / 2 + 1;
        std::vector<q128> g, gw;
        gl_quad(nq, g, gw);
        std::vector<q128> A((size_t)nu * nu, 0), b(nu, 0), P(m + 2);
        for (int q = 0; q < nq; ++q) {
            q128 pm = 1;
            for (int i = 0; i < m; ++i) pm *= g[q] - t[i];
            legendre_all(m + 1, g[q], P.data());
            for (int r = 0; r < nu; ++r) {
                const q128 f = gw[q] * pm * P[2 * r + 1];
                for (int c = 0; c < nu; ++c) A[(size_t)r * nu + c] += f * P[2 * c];
                b[r] -= f * P[m + 1];
            }
        }
        for (int c = 0; c < nu; ++c) {   // Gaussian elimination, partial pivoting
            int piv = c;
            for (int r = c + 1; r < nu; ++r)
                if (fabsq(A[(size_t)r * nu + c]) > fabsq(A[(size_t)piv * nu + c])) piv = r;
            if (piv != c) {
                for (int j = 0; j < nu; ++j) std::swap(A[(size_t)c * nu + j], A[(size_t)piv * nu + j]);
                std::swap(b[c], b[piv]);
            }
            for (int r = c + 1; r < nu; ++r) {
                const q128 f = A[(size_t)r * nu + c] / A[(size_t)c * nu + c];
                for (int j = c; j < nu; ++j) A[(size_t)r * nu + j] -= f * A[(size_t)c * nu + j];
                b[r] -= f * b[c];
            }
        }
        std::vector<q128> a(nu, 0);
        for (int c = nu - 1; c >= 0; --c) {
            q128 v = b[c];
            for (int j = c + 1; j < nu; ++j) v -= A[(size_t)c * nu + j] * a[j];
            a[c] = v / A[(size_t)c * nu + c];
        }
        auto G = [&](q128 x) {
            legendre_all(m + 1, x, P.data());
            q128 v = P[m + 1];
            for (int c = 0; c < nu; ++c) v += a[c] * P[2 * c];
            return v;
        };
        std::vector<q128> nt = t;
        for (int i = 0; i <= m; ++i) {
            q128 lo = i == 0 ? (q128)-1 : t[i - 1], hi = i == m ? (q128)1 : t[i];
            q128 flo = G(lo), fhi = G(hi);
            if (!(flo * fhi < 0)) return false;
            for (int it = 0; it < 200 && hi - lo > 1e-36Q; ++it) {
                const q128 mid = (lo + hi) / 2, fm = G(mid);
                if (fm == 0) {
                    lo = hi = mid;
                    break;
                }
                if ((fm < 0) == (flo < 0)) {
                    lo = mid;
                    flo = fm;
                } else {
                    hi = mid;
                }
            }
            nt.push_back((lo + hi) / 2);
        }
        std::sort(nt.begin(), nt.end());
        t = nt;
    }
    const int n = (int)t.size();
    std::vector<q128> g, gw;
    gl_quad(n / 2 + 2, g, gw);
    wt.assign(n, 0);
    for (int j = 0; j < n; ++j) {
        q128 acc = 0;
        for (size_t q = 0; q < g.size(); ++q) {
            q128 lj = 1;
            for (int i = 0; i < n; ++i)
                if (i != j) lj *= (g[q] - t[i]) / (t[j] - t[i]);
            acc += gw[q] * lj;
        }
        wt[j] = acc;
    }
    return true;
}

// Gauss-Patterson on [0,1] (reading R2): x = (1 + t)/2, w/2; the midpoint is exactly 1/2.
static bool gp_rule_q(int l, double *x, double *w) {
    std::vector<q128> t, wt;
    if (!gp_quad(gp_index(l), t, wt)) return false;
    for (size_t j = 0; j < t.size(); ++j) {
        x[j] = (double)((1 + t[j]) / 2);
        w[j] = (double)(wt[j] / 2);
    }
    return true;
}

int host_rule(int rule, int l, double *x, double *w) {
    int n = host_node_count(rule, l);
    if (n < 0) return -1;
    if (rule == SG_RULE_CLENSHAW_CURTIS) {
        if (l > SG_CC_MAX_LEVEL) return -1;
        cc_rule_q(n, x, w);
    } else if (rule == SG_RULE_TRAPEZOIDAL) {
        if (l > SG_TRAP_MAX_LEVEL) return -1;
        trap_rule_q(n, x, w);
    } else if (rule == SG_RULE_GAUSS_PATTERSON) {
        if (gp_index(l) > SG_GP_MAX_K) return -1;
        if (!gp_rule_q(l, x, w)) return -1;
    } else {
        if (n > SG_GL_MAX_N) return -1;
        gl_rule_q(n, x, w);
    }
    return n;
}

// task descriptor word: two int32 fields (the high one may be negative: source tasks store
// -(k + 1)) packed through unsigned arithmetic; decoded by task_hi32 / task_lo32 (kernels_common.cuh)
static int64_t pack32(int hi, int lo) {
    return (int64_t)(((uint64_t)(uint32_t)hi << 32) | (uint64_t)(uint32_t)lo);
}

static u128 sat_add(u128 a, u128 b) {
    u128 r = a + b;
    const u128 cap = (u128)1 << 100;
    return r > cap ? cap : r;
}
static u128 sat_mul(u128 a, u128 b) {
    const u128 cap = (u128)1 << 100;
    if (a == 0 || b == 0) return 0;
    if (a > cap / b) return cap;
    return a * b;
}

int host_plan_build(HostPlan &hp, int d, int L, int rule, int kind, int form, int merge, int rank, int world,
                    long long range_lo, long long range_hi, int fuse_mode) {
    if (d < 1 || L < 0) return SG_EINVAL;
    if (rule != SG_RULE_CLENSHAW_CURTIS && rule != SG_RULE_GAUSS_LEGENDRE && rule != SG_RULE_TRAPEZOIDAL &&
        rule != SG_RULE_GAUSS_PATTERSON)
        return SG_EINVAL;
    if (kind < 0 || kind > 4 || form < 0 || form > 1 || merge < 0 || merge > 1) return SG_EINVAL;
    hp.merge = merge;
    if (world < 1 || rank < 0 || rank >= world) return SG_EINVAL;
    if (d > SG_MAX_D || L > SG_MAX_L) return SG_EUNSUPPORTED;
    if (rule == SG_RULE_CLENSHAW_CURTIS && L + 1 > SG_CC_MAX_LEVEL) return SG_EUNSUPPORTED;
    if (rule == SG_RULE_TRAPEZOIDAL && L + 1 > SG_TRAP_MAX_LEVEL) return SG_EUNSUPPORTED;
    if (rule == SG_RULE_GAUSS_PATTERSON && gp_index(L + 1) > SG_GP_MAX_K) return SG_EUNSUPPORTED;
    if (rule == SG_RULE_GAUSS_LEGENDRE && L + 1 > SG_GL_MAX_N) return SG_EUNSUPPORTED;
    hp.d = d;
    hp.L = L;
    hp.rule = rule;
    hp.kind = kind;
    hp.form = form;

    // ---- rule entries per level (combination: the level-l rule; delta: Delta^l support) ----
    std::vector<std::vector<double>> RX(L + 2), RW(L + 2);
    for (int l = 1; l <= L + 1; ++l) {
        int n = host_node_count(rule, l);
        RX[l].resize(n);
        RW[l].resize(n);
        if (host_rule(rule, l, RX[l].data(), RW[l].data()) < 0) return SG_EUNSUPPORTED;
    }
    hp.X.clear();
    hp.Whi.clear();
    hp.Wlo.clear();
    // midpoint weight of each level's entries (dd; 0 if the level has no node at 1/2)
    std::vector<double> mid_hi(L + 2, 0.0), mid_lo(L + 2, 0.0);
    int off = 0;
    for (int l = 2; l <= L + 1; ++l) {
        hp.entry_off[l] = off;
        if (form == SG_FORM_COMBINATION) {
            for (size_t j = 0; j < RX[l].size(); ++j) {
                hp.X.push_back(RX[l][j]);
                hp.Whi.push_back(RW[l][j]);
                hp.Wlo.push_back(0.0);
            }
        } else {
            // Delta^l = J^l - J^{l-1} on the union of both node sets; weights as exact dd differences
            std::vector<std::pair<double, std::pair<double, double>>> ent;
            std::vector<bool> used(RX[l - 1].size(), false);
            for (size_t j = 0; j < RX[l].size(); ++j) {
                double wm = 0.0;
                for (size_t i = 0; i < RX[l - 1].size(); ++i)
                    if (RX[l - 1][i] == RX[l][j]) {
                        wm = RW[l - 1][i];
                        used[i] = true;
                    }
                double s = RW[l][j] - wm, bb = s - RW[l][j];
                double e = (RW[l][j] - (s - bb)) + (-wm - bb);
                ent.push_back({RX[l][j], {s, e}});
            }
            for (size_t i = 0; i < RX[l - 1].size(); ++i)
                if (!used[i]) ent.push_back({RX[l - 1][i], {-RW[l - 1][i], 0.0}});
            std::sort(ent.begin(), ent.end(),
                      [](const auto &a, const auto &b) { return a.first < b.first; });
            for (auto &e : ent) {
                hp.X.push_back(e.first);
                hp.Whi.push_back(e.second.first);
                hp.Wlo.push_back(e.second.second);
            }
        }
        // merge: take the midpoint entry out of the level (its copies go into C'(t, b))
        for (size_t i = (size_t)off; i < hp.X.size(); ++i)
            if (hp.X[i] == 0.5) {
                mid_hi[l] = hp.Whi[i];
                mid_lo[l] = hp.Wlo[i];
                if (merge) {
                    hp.X.erase(hp.X.begin() + i);
                    hp.Whi.erase(hp.Whi.begin() + i);
                    hp.Wlo.erase(hp.Wlo.begin() + i);
                }
                break;
            }
        hp.nl[l] = (int)hp.X.size() - off;
        off += hp.nl[l];
    }
    hp.entry_off[L + 2] = off;
    hp.nl[1] = 1;
    hp.M0 = 0;
    for (int l = 2; l <= L + 1; ++l) {
        hp.tab_off[l] = (int)(d * hp.M0);
        hp.M0 += hp.nl[l];
    }
    if ((int64_t)d * hp.M0 > (int64_t)1 << 30) return SG_EUNSUPPORTED;
    hp.tab_entries = (int)(d * hp.M0);
    hp.tab_off[L + 2] = hp.tab_entries;

    // ---- coefficients (Eq 2.6 with q = d + L; delta form: 1) ----
    for (int e = 0; e <= L; ++e) {
        if (form == SG_FORM_DELTA) {
            hp.coef[e] = 1.0;
            continue;
        }
        int m = L - e;
        if (m > d - 1) {
            hp.coef[e] = 0.0;
            continue;
        }
        u128 b = 1;
        for (int i = 1; i <= m; ++i) {
            b = b * (u128)(d - 1 - m + i) / (u128)i;   // exact: C(n-m+i, i) stays integral
            if (b > ((u128)1 << 53)) return SG_EUNSUPPORTED;
        }
        double v = (double)b;
        hp.coef[e] = (m % 2) ? -v : v;
    }

    // ---- node coefficients per (t, b) ----
    hp.cm_hi.assign((size_t)(L + 1) * (L + 1), 0.0);
    hp.cm_lo.assign((size_t)(L + 1) * (L + 1), 0.0);
    for (int t = 0; t <= std::min(L, d); ++t) {
        std::vector<q128> P(L + 1, 0);   // M(z)^(d-t) truncated at z^L, by binary powering
        if (merge) {
            std::vector<q128> Mz(L + 1, 0), B(L + 1, 0), T(L + 1, 0);
            Mz[0] = 1;
            for (int sdeg = 1; sdeg <= L; ++sdeg) Mz[sdeg] = (q128)mid_hi[sdeg + 1] + (q128)mid_lo[sdeg + 1];
            P[0] = 1;
            B = Mz;
            auto mul = [&](const std::vector<q128> &a, const std::vector<q128> &b) {
                std::fill(T.begin(), T.end(), (q128)0);
                for (int i = 0; i <= L; ++i)
                    for (int j = 0; i + j <= L; ++j) T[i + j] += a[i] * b[j];
                return T;
            };
            for (long long n = (long long)d - t; n > 0; n >>= 1) {
                if (n & 1) P = mul(P, B);
                B = mul(B, B);
            }
        }
        for (int b = 0; b <= L; ++b) {
            q128 v = 0;
            if (merge) {
                for (int e = b; e <= L; ++e) v += (q128)hp.coef[e] * P[e - b];
            } else {
                v = hp.coef[b];
            }
            const double hi = (double)v;
            hp.cm_hi[(size_t)t * (L + 1) + b] = hi;
            hp.cm_lo[(size_t)t * (L + 1) + b] = (double)(v - (q128)hi);
        }
    }
    // a node counts as a point iff its coefficient is nonzero (merged: every tree node is a point)
    auto counted = [&](int b) -> bool { return merge || hp.coef[b] != 0.0; };

    hp.maxdepth = std::min(L, d);
    hp.nfront = std::max(0, std::min(L - 1, d - 1));
    const int64_t nd1 = (int64_t)d * hp.M0;

    // ---- subtree point counts Sub[b][k+1] (points with nonzero coefficient) ----
    const int W = d + 1;   // k in [-1, d-1] -> index k+1
    std::vector<u128> Sub((size_t)(L + 1) * W, 0), Suf((size_t)(L + 1) * (W + 1), 0);
    for (int b = L; b >= 0; --b) {
        for (int k = d - 1; k >= -1; --k) {
            u128 s = counted(b) ? 1 : 0;
            for (int lp = 2; lp <= L + 1 - b; ++lp) {
                int bp = b + lp - 1;
                // children at k' > k: Suf[bp][k+1] = sum_{k' >= k+1} Sub[bp][k']
                s = sat_add(s, sat_mul((u128)hp.nl[lp], Suf[(size_t)bp * (W + 1) + (k + 2)]));
            }
            Sub[(size_t)b * W + (k + 1)] = s;
        }
        for (int k = d - 1; k >= -1; --k)
            Suf[(size_t)b * (W + 1) + (k + 1)] =
                sat_add(Suf[(size_t)b * (W + 1) + (k + 2)], Sub[(size_t)b * W + (k + 1)]);
    }
    const u128 total = Sub[0];
    hp.Sub.assign(Sub.size(), 0);
    for (size_t i = 0; i < Sub.size(); ++i)
        hp.Sub[i] = Sub[i] >= ((u128)1 << 63) ? ~(uint64_t)0 : (uint64_t)Sub[i];
    if (total >= ((u128)1 << 63)) return SG_EOVERFLOW;
    hp.total_points = (uint64_t)total;
    const u128 root_w = counted(0) ? 1 : 0;
    auto item_weight = [&](int k1, int l1) -> u128 { return Sub[(size_t)(l1 - 1) * W + (k1 + 1)]; };
    // Shard cost model (balances device time rather than points).  With the last two levels fused
    // (k_leaf2), the subtree of a level-2 depth-1 prefix at coordinate k1 holds
    //   leaf2 = C(d-1-k1, L-1) n2^(L-1)  points evaluated by k_leaf2 (cost 1 each),
    //   mids  = C(d-1-k1, L-2) n2^(L-2)  depth-(L-1) prefixes, each a k_leaf2 row run with a fixed
    //                                     prologue (mid products, bounds, lane fold) ~ LEAF2_MID_COST,
    // and its other points are evaluated by the generic passes at ~GENERIC_POINT_COST each.
    // Measured on config 5 (one B200): k_leaf2 4.6e-13 s/point, k_leaf 8.3e-13 s/point.
    // (depends on the problem's structure only, never on fuse_mode / environment overrides: every
    // rank of a world, and the host-only queries, must cut the same ranges)
    const bool fusable_early = L >= 3 && std::min(L - 1, d - 1) == L - 1 && (hp.nl[2] == 2 || hp.nl[2] == 3);
    auto binom = [](int64_t n, int r) -> double {
        if (r < 0 || n < r) return 0.0;
        double v = 1.0;
        for (int i = 1; i <= r; ++i) v = v * (double)(n - r + i) / (double)i;
        return v;
    };
    double cost_generic = GENERIC_POINT_COST, cost_mid = LEAF2_MID_COST;
    if (const char *e = getenv("SG_B200_COST_GENERIC"); e && e[0]) cost_generic = atof(e);   // A/B runs
    if (const char *e = getenv("SG_B200_COST_MID"); e && e[0]) cost_mid = atof(e);
    auto item_cost = [&](int k1, int l1) -> double {
        const double pts = (double)item_weight(k1, l1);
        if (!fusable_early || l1 != 2) return cost_generic * pts;
        const double n2 = (double)hp.nl[2];
        const double leaf2 = binom(d - 1 - k1, L - 1) * std::pow(n2, L - 1);
        const double mids = binom(d - 1 - k1, L - 2) * std::pow(n2, L - 2);
        return leaf2 + cost_generic * std::max(0.0, pts - leaf2) + cost_mid * mids;
    };

    // ---- shard range in depth-1 rank space ----
    int64_t lo = 0, hi = nd1;
    const bool explicit_range = range_hi > range_lo && range_lo >= 0;
    if (explicit_range) {
        lo = std::min<int64_t>(range_lo, nd1);
        hi = std::min<int64_t>(range_hi, nd1);
    } else if (world > 1) {
        // cut points by the cost model above (double precision is ample: only balance depends on
        // it; the points each rank evaluates are counted exactly below)
        double total_cost = (double)root_w;
        for (int k1 = 0; k1 < d; ++k1)
            for (int l1 = 2; l1 <= L + 1; ++l1) total_cost += hp.nl[l1] * item_cost(k1, l1);
        auto cut = [&](int r) -> int64_t {
            if (r <= 0) return 0;
            if (r >= world) return nd1;
            const double target = total_cost * (double)r / (double)world;
            double cum = (double)root_w;
            if (cum >= target) return 0;
            int64_t pos = 0;
            for (int k1 = 0; k1 < d; ++k1)
                for (int l1 = 2; l1 <= L + 1; ++l1) {
                    const double wgt = item_cost(k1, l1), n = (double)hp.nl[l1];
                    if (wgt > 0.0 && cum + n * wgt >= target) {
                        const int64_t take = (int64_t)std::ceil((target - cum) / wgt);
                        return pos + std::min<int64_t>(std::max<int64_t>(take, 0), hp.nl[l1]);
                    }
                    cum += n * wgt;
                    pos += hp.nl[l1];
                }
            return nd1;
        };
        lo = cut(rank);
        hi = cut(rank + 1);
    }
    hp.range_lo = lo;
    hp.range_hi = hi;
    // the root point belongs to exactly one shard: rank 0 of a world partition (cut() may give
    // several ranks an empty range starting at 0), or an explicit range that starts at 0
    hp.include_root = explicit_range ? (lo == 0) : (rank == 0);
    {
        u128 sp = hp.include_root ? root_w : 0;
        int64_t pos = 0;
        for (int k1 = 0; k1 < d; ++k1)
            for (int l1 = 2; l1 <= L + 1; ++l1) {
                int64_t a = std::max<int64_t>(lo, pos), b = std::min<int64_t>(hi, pos + hp.nl[l1]);
                if (b > a) sp += (u128)(b - a) * item_weight(k1, l1);
                pos += hp.nl[l1];
            }
        hp.shard_points = (uint64_t)sp;
    }

    // ---- frontier counts ----
    const size_t LD = (size_t)std::max(L, 1) * d;
    hp.N.assign(hp.nfront + 2, std::vector<int64_t>());
    hp.C.assign(hp.nfront + 2, std::vector<int64_t>());
    hp.off.assign(hp.nfront + 2, std::vector<int64_t>());
    hp.total.assign(hp.nfront + 2, 0);
    hp.TB.assign(hp.nfront + 2, std::vector<int64_t>());
    hp.JS.assign(LD, 0);
    auto finish_depth = [&](int t) -> int {
        std::vector<int64_t> &N = hp.N[t], &C = hp.C[t], &O = hp.off[t];
        C.assign(LD, 0);
        O.assign(LD, 0);
        u128 run = 0;
        for (int b = 0; b < L; ++b) {
            int64_t c = 0;
            for (int k = 0; k < d; ++k) {
                C[(size_t)b * d + k] = c;
                c += N[(size_t)b * d + k];
                O[(size_t)b * d + k] = (int64_t)run;
                run += (u128)N[(size_t)b * d + k];
                if (run >= ((u128)1 << 62)) return SG_EOVERFLOW;
            }
        }
        hp.total[t] = (int64_t)run;
        return SG_OK;
    };
    if (hp.nfront >= 1) {
        hp.N[1].assign(LD, 0);
        int64_t pos = 0;
        for (int k1 = 0; k1 < d; ++k1)
            for (int l1 = 2; l1 <= L + 1; ++l1) {
                int b = l1 - 1;
                int64_t a = std::max<int64_t>(lo, pos), e = std::min<int64_t>(hi, pos + hp.nl[l1]);
                if (e > a && b <= L - 1 && k1 <= d - 2) {
                    hp.N[1][(size_t)b * d + k1] = e - a;
                    hp.JS[(size_t)b * d + k1] = a - pos;
                }
                pos += hp.nl[l1];
            }
        int rc = finish_depth(1);
        if (rc) return rc;
        for (int t = 1; t < hp.nfront; ++t) {
            std::vector<int64_t> &Nn = hp.N[t + 1];
            Nn.assign(LD, 0);
            for (int bp = t + 1; bp <= L - 1; ++bp)
                for (int kp = 0; kp <= d - 2; ++kp) {
                    u128 s = 0;
                    for (int b = 0; b < bp; ++b)
                        s += (u128)hp.nl[bp - b + 1] * (u128)hp.C[t][(size_t)b * d + kp];
                    if (s >= ((u128)1 << 62)) return SG_EOVERFLOW;
                    Nn[(size_t)bp * d + kp] = (int64_t)s;
                }
            rc = finish_depth(t + 1);
            if (rc) return rc;
            std::vector<int64_t> &T = hp.TB[t];
            T.assign((size_t)L * L * d, 0);
            for (int bp = t + 1; bp <= L - 1; ++bp)
                for (int kp = 0; kp < d; ++kp) {
                    int64_t acc = hp.off[t + 1][(size_t)bp * d + kp];
                    for (int b = 0; b < bp; ++b) {
                        T[((size_t)b * L + bp) * d + kp] = acc;
                        acc += (int64_t)hp.nl[bp - b + 1] * hp.C[t][(size_t)b * d + kp];
                    }
                }
        }
    }

    // ---- pass statistics and launch geometry ----
    const int64_t WARPS_PER_BLOCK = 8, TARGET_WARPS = 148 * 64;
    hp.pass_terms.assign(hp.nfront + 1, 0);
    hp.pass_written.assign(hp.nfront + 1, 0);
    hp.pass_nsplit.assign(hp.nfront + 1, 1);
    hp.pass_ntasks.assign(hp.nfront + 1, 0);
    hp.pass_blocks.assign(hp.nfront + 1, 0);
    hp.pass_partial_off.assign(hp.nfront + 1, 0);
    hp.pass_terms[0] = (uint64_t)(hi - lo);
    hp.pass_written[0] = hp.nfront >= 1 ? (uint64_t)hp.total[1] : 0;
    // root partial slots: one per 256 depth-1 prefixes of the WHOLE rank space, i.e. one per K0 block
    // (k_head computes each depth-1 point in the K0 thread of its factor entry; the separate k_root
    // launches the same number of blocks, those past the shard range write zero)
    hp.root_blocks = std::max<int64_t>(1, (nd1 + 255) / 256);
    int64_t poff = hp.root_blocks;
    for (int t = 1; t <= hp.nfront; ++t) {
        u128 terms = 0;
        for (int b = 0; b < L; ++b) {
            int64_t ml = 0;
            for (int lp = 2; lp <= L + 1 - b; ++lp) ml += hp.nl[lp];
            for (int k = 0; k < d; ++k)
                terms += (u128)hp.N[t][(size_t)b * d + k] * (u128)(d - 1 - k) * (u128)ml;
        }
        hp.pass_terms[t] = (uint64_t)terms;
        hp.pass_written[t] = (t + 1 <= hp.nfront) ? (uint64_t)hp.total[t + 1] : 0;
        int64_t chunks = (hp.total[t] + 31) / 32;
        int64_t ns = chunks > 0 ? (TARGET_WARPS + chunks - 1) / chunks : 1;
        ns = std::max<int64_t>(1, std::min<int64_t>(ns, d));
        hp.pass_nsplit[t] = (int)ns;
        hp.pass_ntasks[t] = chunks * ns;
        hp.pass_blocks[t] = std::max<int64_t>(1, (hp.pass_ntasks[t] + WARPS_PER_BLOCK - 1) / WARPS_PER_BLOCK);
        hp.pass_partial_off[t] = poff;
        poff += hp.pass_blocks[t];
    }
    hp.total_partials = poff;
    // ---- fused last two levels ----
    // fused whenever possible (measured: config 5 30.25 -> 27.55 ms, config 4 2.43 -> 2.19 ms with
    // the NJ-mid-parallel k_leaf2); fuse_mode 0 keeps the stored frontier (A/B, tests)
    const bool fusable = L >= 3 && hp.nfront == L - 1 && (hp.nl[2] == 2 || hp.nl[2] == 3);
    hp.fuse = fusable && fuse_mode != 0;
    if (hp.fuse) {
        const int tm = L - 2;   // depth of the stored parents; their excess is L-2
        hp.pass_written[tm] = 0;
        // Cmid[k] = parents (excess L-2) whose last active coordinate is < k; chunk c of 32 parents
        // has a valid lane for every k_mid >= kstart(c) (Cmid is nondecreasing); k_mid <= d-2
        auto cmid = [&](int k) -> int64_t { return k <= d - 2 ? hp.C[tm][(size_t)(L - 2) * d + k] : 0; };
        // a level-2 row that is one conjugate pair (oscillatory, x_0 = 1 - x_1, equal weights:
        // the midpoint-merged CC row) runs k_leaf2_pairs with LEAF2_PPL parents per lane
        {
            const int e0 = hp.entry_off[2];
            const bool pair = kind == SG_F_OSCILLATORY && hp.nl[2] == 2 && 1.0 - hp.X[e0 + 1] == hp.X[e0] &&
                              hp.Whi[e0] == hp.Whi[e0 + 1] && hp.Wlo[e0] == hp.Wlo[e0 + 1];
            const bool sym3 = kind == SG_F_OSCILLATORY && hp.nl[2] == 3 && hp.X[e0 + 1] == 0.5 &&
                              1.0 - hp.X[e0 + 2] == hp.X[e0] && hp.Whi[e0] == hp.Whi[e0 + 2] &&
                              hp.Wlo[e0] == hp.Wlo[e0 + 2];
            hp.leaf2_ppl = pair ? LEAF2_PPL : sym3 ? LEAF2_PPL3 : 1;
            hp.leaf2_sym3 = sym3 && !pair;
        }
        // Lane groups (real kinds, one parent per lane): with few parents (a small shard) the last
        // chunk of 32 is mostly empty lanes (config 4, rank 0 of 8: 132 parents -> 0.82 of the lanes
        // busy); 32 / G parents per chunk and G k_mid groups per warp fill them.  The smallest G whose
        // lane fill is >= 0.97 (1 on every full-size problem; the plan depends on the problem and
        // the shard only, so every rank and the host queries agree).
        hp.leaf2_groups = 1;
        if (kind != SG_F_OSCILLATORY && hp.leaf2_ppl == 1) {
            const int64_t np = cmid(d - 2);
            auto fill = [&](int g) {
                const int64_t pc = 32 / g;
                return np > 0 ? (double)np / (double)(((np + pc - 1) / pc) * pc) : 1.0;
            };
            int best = 1;
            for (int g : {1, 2, 4, 8}) {
                if (fill(g) >= 0.97) {
                    best = g;
                    break;
                }
                if (fill(g) > fill(best) + 1e-9) best = g;
            }
            if (const char *e = getenv("SG_B200_LEAF2_GROUPS"); e && e[0]) best = atoi(e);   // A/B runs
            if (best == 1 || best == 2 || best == 4 || best == 8) hp.leaf2_groups = best;
        }
        const int G = hp.leaf2_groups;
        const int64_t CH = 32LL * hp.leaf2_ppl / G;   // parents per task chunk
        const int64_t nchunks = (cmid(d - 2) + CH - 1) / CH;
        struct Task {
            int64_t rows, first;
            int ka, kb, kp0, kp1;   // k_mid range; row range (split tasks: one k_mid block, [kp0, kp1))
        };
        std::vector<Task> tasks;
        int k0 = 0;
        for (int64_t c = 0; c < nchunks; ++c) {
            while (k0 <= d - 2 && cmid(k0) <= CH * c) ++k0;   // kstart(c), nondecreasing in c
            if (G == 1) {
                int64_t acc = 0;
                int ka = k0;
                for (int k = k0; k <= d - 2; ++k) {
                    acc += d - 1 - k;
                    if (acc >= LEAF2_TASK_ROWS || k == d - 2) {
                        tasks.push_back(Task{acc, CH * c, ka, k + 1, 0, d});
                        acc = 0;
                        ka = k + 1;
                    }
                }
                continue;
            }
            // G > 1: blocks of G consecutive k_mids (one per lane group), grouped until the first
            // group's rows (the longest) reach LEAF2_TASK_ROWS; rows = that group's row count
            for (int km = k0; km <= d - 2;) {
                const int ka = km;
                int64_t grows = 0;
                while (km <= d - 2 && grows < LEAF2_TASK_ROWS) {
                    grows += d - 1 - km;
                    km += G;
                }
                tasks.push_back(Task{grows, CH * c, ka, std::min(km, d - 1), 0, d});
            }
        }
        // Source tasks (k_leaf2_sym3 plans whose level 3 has SYM3_N3 nodes): pass L-2 runs
        // k_leaf2_sym3<SRC = true> over every source of frontier L-2 instead of k_leaf.  A task is a
        // chunk of 32 * 3 * PPL sources with the same last active coordinate k (one prefix per lane
        // and accumulator slot): the excess-(L-1) sources' symmetric level-2 rows k' = k+1 .. d-1,
        // the excess-(L-2) sources' level-2 rows (coefficient coef[L-1], SRC_CPREV) and their
        // level-3 rows (SRC_L3).  Encoded with ka = -(k + 1), kb = chunk size | flags; heavy-first,
        // never split (rows <= d - 1); one partial slot per task.
        std::vector<Task> srct;
#ifndef LEAF2_NO_SRCTASKS
        if (hp.leaf2_sym3 && L >= 3 && merge == 0 && hp.nl[3] == SYM3_N3) {
            const int64_t CHB = 32LL * 3 * hp.leaf2_ppl;
            // task weight = rows (level-3 rows: 3 rows); when the longest task exceeds one resident
            // warp's share of the total (a small shard), rows are split into pieces of about half a
            // share (measured, config 5 unsplit at N = 1 and split at N = 8: 0.43 / ~0.06 ms)
            double wsum = 0.0, wmax = 0.0;
            for (int b = L - 2; b <= L - 1; ++b)
                for (int k = 0; k <= d - 2; ++k) {
                    const int64_t chunks = (hp.N[tm][(size_t)b * d + k] + CHB - 1) / CHB;
                    const double w = (double)(d - 1 - k) * (b == L - 1 ? 1.0 : 4.0);
                    wsum += (double)chunks * w;
                    if (chunks > 0) wmax = std::max(wmax, (double)(d - 1 - k) * (b == L - 1 ? 1.0 : 3.0));
                }
            const double share = wsum / (double)SYM3_RESIDENT_WARPS;
            int rmax = d;   // rows per piece (weight-1 rows; level-3 pieces get a third)
            if (LEAF2_SRC_ROWS > 0) rmax = LEAF2_SRC_ROWS;
            else if (wmax > share) rmax = std::max(8, (int)(share / 2.0));
            for (int b = L - 2; b <= L - 1; ++b)
                for (int k = 0; k <= d - 2; ++k) {
                    const int64_t n = hp.N[tm][(size_t)b * d + k], o = hp.off[tm][(size_t)b * d + k];
                    const int rows = d - 1 - k;
                    // level-2 pieces of <= rmax rows; the level-3 tasks of excess-(L-2) sources use
                    // pieces of <= rmax / 3 rows (their rows cost three level-2 rows)
                    const int r2 = rmax, r3 = rmax >= d ? d : std::max(4, rmax / 3);
                    const int pieces = b == L - 1 ? (rows + r2 - 1) / r2 : (rows + r3 - 1) / r3;
                    for (int64_t c = 0; c < n; c += CHB)
                        for (int q = 0; q < pieces; ++q) {
                            const int cnt = (int)std::min<int64_t>(CHB, n - c);
                            const int a0 = k + 1 + (int)((int64_t)rows * q / pieces);
                            const int a1 = k + 1 + (int)((int64_t)rows * (q + 1) / pieces);
                            if (b == L - 1) {
                                srct.push_back(Task{a1 - a0, o + c, -(k + 1), cnt, a0, a1});
                            } else {
                                srct.push_back(Task{a1 - a0, o + c, -(k + 1), cnt | SRC_CPREV, a0, a1});
                                srct.push_back(Task{3LL * (a1 - a0), o + c, -(k + 1), cnt | SRC_L3, a0, a1});
                            }
                        }
                }
            hp.leaf2_srctasks = true;
            std::stable_sort(srct.begin(), srct.end(), [](const Task &a, const Task &b) {
                if (a.rows != b.rows) return a.rows > b.rows;
                if (a.ka != b.ka) return a.ka < b.ka;
                if (a.kb != b.kb) return a.kb < b.kb;
                if (a.first != b.first) return a.first < b.first;
                return a.kp0 < b.kp0;
            });
            hp.T2S.resize(3 * srct.size());
            for (size_t i = 0; i < srct.size(); ++i) {
                hp.T2S[3 * i] = srct[i].first;
                hp.T2S[3 * i + 1] = pack32(srct[i].ka, srct[i].kb);
                hp.T2S[3 * i + 2] = pack32(srct[i].kp0, srct[i].kp1);
            }
            hp.pass_nsplit[tm] = 1;
            hp.pass_ntasks[tm] = (int64_t)srct.size();
            hp.pass_blocks[tm] = (int64_t)srct.size();   // one partial slot per task
        }
#endif
        // When the longest task is a large share of one resident warp's work (a small shard: config 4
        // on 8 GPUs), the persistent grid's tail is a handful of long single-k_mid tasks: split
        // their rows into pieces of LEAF2_TASK_ROWS (partials stay per task, order fixed).
        int64_t total_rows = 0, max_rows = 0;
        for (const Task &tk : tasks) {
            total_rows += tk.rows;
            max_rows = std::max(max_rows, tk.rows);
        }
        const bool do_split =
            max_rows > LEAF2_TASK_ROWS && LEAF2_SPLIT_SHARE * max_rows * (int64_t)LEAF2_RESIDENT_WARPS > total_rows;
        // piece length: about LEAF2_PIECES_PER_WARP pieces per resident warp (the dynamic schedule's
        // tail is about one piece), at most LEAF2_TASK_ROWS and at least LEAF2_MIN_PIECE rows (each
        // piece repeats its k_mid prologue)
        int64_t ppw = LEAF2_PIECES_PER_WARP;
        if (const char *e = getenv("SG_B200_PIECES"); e && e[0]) ppw = std::max(1, atoi(e));   // A/B runs
        const int64_t piece = std::max<int64_t>(
            LEAF2_MIN_PIECE, std::min<int64_t>(LEAF2_MAX_PIECE, total_rows / ((int64_t)LEAF2_RESIDENT_WARPS * ppw)));
        if (do_split) {
            std::vector<Task> split;
            for (const Task &tk : tasks) {
                if (tk.kb - tk.ka > G || tk.rows <= piece) {   // one k_mid block only
                    split.push_back(tk);
                    continue;
                }
                const int pieces = (int)((tk.rows + piece - 1) / piece);
                const int r0 = tk.ka + 1;
                for (int q = 0; q < pieces; ++q) {
                    const int a = r0 + (int)((int64_t)tk.rows * q / pieces);
                    const int b = r0 + (int)((int64_t)tk.rows * (q + 1) / pieces);
                    split.push_back(Task{b - a, tk.first, tk.ka, tk.kb, a, b});
                }
            }
            tasks.swap(split);
        }
        if (const char *dbg = getenv("SG_B200_DEBUG_TASKS"); dbg && dbg[0] == '1') {
            // lane utilisation: parent-rows with a valid lane / lane-row slots the tasks occupy
            double useful = 0, slots = 0, tail = 0;
            for (int k = 0; k + 1 <= d - 2; ++k) {
                tail = 0;
                for (int km = k + 1; km <= d - 2; ++km) tail += d - 1 - km;
                useful += (double)(cmid(k + 1) - cmid(k)) * tail;
            }
            for (const Task &tk : tasks) slots += (double)tk.rows * CH * G;
            fprintf(stderr, "leaf2 tasks: %zu total_rows %lld max_rows %lld split %d ppl %d parents %lld "
                    "lane_util %.4f groups %d\n", tasks.size(), (long long)total_rows, (long long)max_rows, (int)do_split,
                    hp.leaf2_ppl, (long long)cmid(d - 2), useful / slots, G);
        }
        // task cost for the schedule: rows + LEAF2_PRO_COST per k_mid block (its prologue: the
        // mid products, grid bounds and lane epilogue, about two rows' work)
        auto tcost = [G](const Task &tk) -> int64_t {
            return tk.rows + (int64_t)LEAF2_PRO_COST * ((tk.kb - tk.ka + G - 1) / G);
        };
        // heavy-first (by cost) for the dynamic scheduler; ties in a fixed order (k_mid, rows, chunk)
        std::stable_sort(tasks.begin(), tasks.end(), [&tcost](const Task &a, const Task &b) {
            const int64_t ca = tcost(a), cb = tcost(b);
            if (ca != cb) return ca > cb;
            if (a.rows != b.rows) return a.rows > b.rows;
            if (a.ka != b.ka) return a.ka < b.ka;
            if (a.kp0 != b.kp0) return a.kp0 < b.kp0;
            return a.first < b.first;
        });
        // Guided tail (guided self-scheduling on the fixed list): a task claimed when work W_rem
        // (itself and everything after it) is left is cut to at most LEAF2_GUIDE x W_rem / resident
        // warps rows (>= LEAF2_MIN_PIECE), so the tasks in flight when the list runs dry are short.
        // Measured (tools/tail_profile.py, config 4): without it the warps exit over the last 8% of
        // the launch at N = 1 and 25% at N = 8 — the youngest CTA of each SM is starved by the
        // scheduler's age priority and still holds a full task when the list empties.  Single-k_mid
        // tasks split by rows, grouped tasks by k_mid blocks; pieces stay in list order.
        if (LEAF2_GUIDE > 0.0) {
            double guide = LEAF2_GUIDE;
            if (const char *e = getenv("SG_B200_GUIDE"); e && e[0]) guide = atof(e);   // A/B runs
            int64_t gmin = LEAF2_GUIDE_MIN;
            if (const char *e = getenv("SG_B200_GUIDE_MIN"); e && e[0]) gmin = std::max(1, atoi(e));   // A/B runs
            // resident warps of the kernel that runs the list: 8 / SM (k_leaf2_sym3, k_leaf2_pairs:
            // one 8-warp CTA), 16 (k_leaf2, oscillatory), 24 (k_leaf2, real kinds)
            const double W = hp.leaf2_ppl > 1 ? 148.0 * 8 : kind == SG_F_OSCILLATORY ? 148.0 * 16 : 148.0 * 24;
            std::vector<Task> rev;
            rev.reserve(tasks.size() + tasks.size() / 4);
            double rem = 0.0;
            for (size_t ii = tasks.size(); ii-- > 0;) {
                const Task &tk = tasks[ii];
                rem += (double)tcost(tk);
                const int64_t cap = std::max<int64_t>(gmin, (int64_t)(guide * rem / W));
                if (guide <= 0.0 || tcost(tk) <= cap) {
                    rev.push_back(tk);
                    continue;
                }
                std::vector<Task> pcs;
                if (tk.kb - tk.ka <= G) {
                    // one k_mid block: rows [max(ka + 1, kp0), kp1) of its first group in pieces
                    const int r0 = std::max(tk.ka + 1, tk.kp0), r1 = std::min(tk.kp1, d);
                    const int nr = r1 - r0;
                    const int64_t rcap = std::max<int64_t>(1, cap - LEAF2_PRO_COST);
                    const int pieces = (int)std::min<int64_t>(nr, (nr + rcap - 1) / rcap);
                    for (int q = 0; q < pieces; ++q) {
                        const int a = r0 + (int)((int64_t)nr * q / pieces);
                        const int b = r0 + (int)((int64_t)nr * (q + 1) / pieces);
                        pcs.push_back(Task{b - a, tk.first, tk.ka, tk.kb, a, b});
                    }
                } else {
                    // k_mid blocks of G (the first group's rows d - 1 - km per block), cut greedily
                    // without overshooting the cap: a piece closes before the block that would take
                    // it past the cap, and a block longer than the cap on its own is cut into row
                    // pieces (every lane group walks the same row range [kp0, kp1))
                    int ka = tk.ka;
                    int64_t acc = 0;
                    int64_t accc = 0;   // acc in cost units
                    for (int km = tk.ka; km < tk.kb; km += G) {
                        const int64_t r = d - 1 - km;
                        const int nx = std::min(km + G, tk.kb);
                        if (acc > 0 && accc + r + LEAF2_PRO_COST > cap) {
                            pcs.push_back(Task{acc, tk.first, ka, km, tk.kp0, tk.kp1});
                            acc = accc = 0;
                            ka = km;
                        }
                        if (r + LEAF2_PRO_COST > cap && tk.kp0 == 0 && tk.kp1 == d) {
                            const int r0 = km + 1, nr = (int)r;
                            const int64_t rcap = std::max<int64_t>(1, cap - LEAF2_PRO_COST);
                            const int pieces = (int)std::min<int64_t>(nr, (nr + rcap - 1) / rcap);
                            for (int q = 0; q < pieces; ++q) {
                                const int a = r0 + (int)((int64_t)nr * q / pieces);
                                const int b = r0 + (int)((int64_t)nr * (q + 1) / pieces);
                                pcs.push_back(Task{b - a, tk.first, km, nx, a, b});
                            }
                            ka = nx;
                            continue;
                        }
                        acc += r;
                        accc += r + LEAF2_PRO_COST;
                        if (accc >= cap || nx >= tk.kb) {
                            pcs.push_back(Task{acc, tk.first, ka, nx, tk.kp0, tk.kp1});
                            acc = accc = 0;
                            ka = nx;
                        }
                    }
                }
                for (size_t q = pcs.size(); q-- > 0;) rev.push_back(pcs[q]);
            }
            tasks.assign(rev.rbegin(), rev.rend());
        }
        if (const char *dbg = getenv("SG_B200_DEBUG_TASKS"); dbg && dbg[0] == '1') {
            // list schedule of the sorted tasks on the resident warps (cost = rows + 2 per k_mid of the
            // task's group for its prologue): makespan against the perfect balance (tail loss)
            std::vector<double> wq(LEAF2_RESIDENT_WARPS, 0.0);
            std::make_heap(wq.begin(), wq.end(), std::greater<double>());
            double tot = 0.0;
            for (const Task &tk : tasks) {
                const double c = (double)tcost(tk);
                std::pop_heap(wq.begin(), wq.end(), std::greater<double>());
                wq.back() += c;
                std::push_heap(wq.begin(), wq.end(), std::greater<double>());
                tot += c;
            }
            const double mk = *std::max_element(wq.begin(), wq.end());
            fprintf(stderr, "leaf2 schedule: makespan %.0f avg %.0f efficiency %.4f\n", mk,
                    tot / LEAF2_RESIDENT_WARPS, tot / LEAF2_RESIDENT_WARPS / mk);
        }
        if (const char *fn = getenv("SG_B200_DUMP_TASKS"); fn && fn[0]) {
            // the fused task list in claim order (tests: coverage of every (chunk, k_mid, row) once)
            if (FILE *f = fopen(fn, "w")) {
                fprintf(f, "%d %d %d\n", G, d, (int)CH);
                for (const Task &tk : tasks)
                    fprintf(f, "%lld %lld %d %d %d %d\n", (long long)tk.rows, (long long)tk.first, tk.ka, tk.kb,
                            tk.kp0, tk.kp1);
                fclose(f);
            }
        }
        hp.T2.resize(3 * tasks.size());
        for (size_t i = 0; i < tasks.size(); ++i) {
            hp.T2[3 * i] = tasks[i].first;
            hp.T2[3 * i + 1] = pack32(tasks[i].ka, tasks[i].kb);
            hp.T2[3 * i + 2] = pack32(tasks[i].kp0, tasks[i].kp1);
        }
        const int t = hp.nfront;
        hp.pass_nsplit[t] = 1;
        hp.pass_ntasks[t] = (int64_t)tasks.size();
        hp.pass_blocks[t] = std::max<int64_t>(1, (hp.pass_ntasks[t] + WARPS_PER_BLOCK - 1) / WARPS_PER_BLOCK);
        poff = hp.root_blocks;
        for (int u = 1; u <= hp.nfront; ++u) {
            hp.pass_partial_off[u] = poff;
            poff += hp.pass_blocks[u];
        }
        hp.total_partials = poff;
    }
    const bool cplx = (kind == SG_F_OSCILLATORY);
    const size_t per_node = (cplx ? 32 : 16) + 4;
    for (int par = 0; par < 2; ++par) {
        int64_t cap = 0;
        for (int t = 1; t <= hp.nfront; ++t)
            if (t % 2 == par && !(hp.fuse && t == hp.nfront)) cap = std::max(cap, hp.total[t]);
        cap = (cap + 63) / 64 * 64;
        hp.ws_front_cap[par] = cap;
        hp.ws_front_bytes[par] = (size_t)cap * per_node;
    }
    return SG_OK;
}

int host_unrank(const HostPlan &hp, uint64_t index, int *t, int *k, int *l, int *j, double *coef) {
    if (index >= hp.shard_points) return SG_EINVAL;
    const int d = hp.d, L = hp.L, W = d + 1;
    auto sub = [&](int b, int kk) -> uint64_t { return hp.Sub[(size_t)b * W + (kk + 1)]; };
    uint64_t r = index;
    int depth = 0, b = 0, kl = -1;
    // root
    auto counted = [&](int bb) -> bool { return hp.merge || hp.coef[bb] != 0.0; };
    if (hp.include_root && counted(0)) {
        if (r == 0) {
            *t = 0;
            *coef = hp.cm_hi[0];
            return SG_OK;
        }
        r -= 1;
    }
    // depth-1 subtrees of the shard's r1 range
    bool found = false;
    int64_t pos = 0;
    for (int k1 = 0; k1 < d && !found; ++k1)
        for (int l1 = 2; l1 <= L + 1 && !found; ++l1) {
            const int64_t a = std::max<int64_t>(hp.range_lo, pos), e = std::min<int64_t>(hp.range_hi, pos + hp.nl[l1]);
            if (e > a) {
                const uint64_t s = sub(l1 - 1, k1);
                const uint64_t blk = (uint64_t)(e - a) * s;
                if (r < blk) {
                    const int j1 = (int)(a - pos + (int64_t)(r / s));
                    r %= s;
                    k[0] = k1;
                    l[0] = l1;
                    j[0] = j1;
                    depth = 1;
                    b = l1 - 1;
                    kl = k1;
                    found = true;
                } else {
                    r -= blk;
                }
            }
            pos += hp.nl[l1];
        }
    if (!found) return SG_EINVAL;
    // descend in preorder
    for (;;) {
        if (counted(b)) {
            if (r == 0) break;
            r -= 1;
        }
        bool moved = false;
        for (int kp = kl + 1; kp < d && !moved; ++kp)
            for (int lp = 2; lp <= L + 1 - b && !moved; ++lp) {
                const uint64_t s = sub(b + lp - 1, kp);
                const uint64_t blk = (uint64_t)hp.nl[lp] * s;
                if (r < blk) {
                    k[depth] = kp;
                    l[depth] = lp;
                    j[depth] = (int)(r / s);
                    r %= s;
                    ++depth;
                    b += lp - 1;
                    kl = kp;
                    moved = true;
                } else {
                    r -= blk;
                }
            }
        if (!moved) return SG_EINVAL;   // inconsistent counts (cannot happen for a valid plan)
    }
    *t = depth;
    *coef = hp.cm_hi[(size_t)depth * (L + 1) + b];
    return SG_OK;
}
