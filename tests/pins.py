"""Independent high-precision pins (test-side, mpmath).  Shares no code with oracle/ or the CUDA path.

* ``mp_rule``         — the paper's 1-D rules evaluated in mpmath and rounded
                         to float64; used to check the oracle's tables bit-for-bit (pin P4).
* ``dp_value``        — the exact Smolyak sum A(d+L, d) for product-form integrands by the
                         generating-function identity  sum_{|i|=d+e} prod_k J^{i_k}(g_k)
                         = [z^e] prod_k (sum_l J^l(g_k) z^{l-1})  (distributivity applied to
                         PAPER.md:67 Eq 2.6 / :71 Eq 2.7; SURVEY.md §8c pin P1).  O(d L^2).
* ``closed_form``     — the exact integral on [0,1]^d (BASELINE.json configs; pin P7).
"""
from __future__ import annotations

import functools

import mpmath as mp

import sg_configs as S

DPS = 50


@functools.lru_cache(maxsize=None)
def mp_rule(rule: int, level: int):
    """(nodes, weights) as float64 tuples, from 50-digit evaluations of the paper's formulas."""
    with mp.workdps(DPS):
        if rule == S.RULE_CC:
            n = 1 if level == 1 else 2 ** (level - 1) + 1
            if n == 1:
                return (0.5,), (1.0,)
            m = n - 1
            xs, ws = [], []
            for j in range(1, n + 1):
                x = -mp.cos(mp.pi * (j - 1) / m)
                if j in (1, n):
                    wt = mp.mpf(1) / (n * (n - 2))
                else:
                    s = mp.mpf(0)
                    for k in range(1, m // 2 + 1):
                        t = mp.cos(2 * mp.pi * (j - 1) * k / m) / (1 - 4 * k * k)
                        if k == m // 2:
                            t /= 2
                        s += t
                    wt = mp.mpf(2) / m * (1 + 2 * s)
                xs.append(float((x + 1) / 2))
                ws.append(float(wt / 2))
            return tuple(xs), tuple(ws)
        if rule == S.RULE_GL:
            n = level
            if n == 1:
                return (0.5,), (1.0,)
            # roots of P_n via mpmath's polyroots on the explicit Legendre coefficients
            coeffs = mp.taylor(lambda t: mp.legendre(n, t), 0, n)[::-1]
            roots = sorted(mp.re(r) for r in mp.polyroots(coeffs, maxsteps=400, extraprec=400))
            xs, ws = [], []
            for t in roots:
                dp = mp.diff(lambda s: mp.legendre(n, s), t)
                wt = 2 / ((1 - t * t) * dp * dp)
                xs.append(float((1 + t) / 2))
                ws.append(float(wt / 2))
            return tuple(xs), tuple(ws)
        if rule == S.RULE_TRAP:
            # Eq 2.10 on [-1,1]: x_j = (j-1) 2^{2-l} - 1, w = 2^{2-l}, ends halved; mapped to [0,1]
            if level == 1:
                return (0.5,), (1.0,)
            n = 2 ** (level - 1) + 1
            h = mp.mpf(2) ** (2 - level)
            xs = [float(((j - 1) * h - 1 + 1) / 2) for j in range(1, n + 1)]
            ws = [float((h / 2 if j in (1, n) else h) / 2) for j in range(1, n + 1)]
            return tuple(xs), tuple(ws)
        if rule == S.RULE_GP:
            t, w = _mp_patterson(gp_extensions(level))
            return tuple(float((1 + a) / 2) for a in t), tuple(float(b / 2) for b in w)
    raise ValueError(rule)


def gp_extensions(level: int) -> int:
    """Patterson extensions for Gauss-Patterson level l: the first rule (2^{i+1}-1 points, degree of
    exactness 1 or 3*2^i - 1) exact to the degree 2l-1 of the l-point Gauss rule (PAPER.md:615
    sequence 1, 3, 3, 7, 7, 7, 15, ...)."""
    i = 0
    while (1 if i == 0 else 3 * 2 ** i - 1) < 2 * level - 1:
        i += 1
    return i


def _mp_legendre_all(n, x):
    P = [mp.mpf(1), x]
    for k in range(2, n + 1):
        P.append(((2 * k - 1) * x * P[-1] - (k - 1) * P[-2]) / k)
    return P[:n + 1]


@functools.lru_cache(maxsize=None)
def _mp_gauss(n):
    """n-point Gauss-Legendre on [-1,1] at the working precision (Newton on P_n)."""
    xs, ws = [], []
    for i in range(1, n + 1):
        x = mp.cos(mp.pi * (i - mp.mpf(0.25)) / (n + mp.mpf(0.5)))
        for _ in range(200):
            P = _mp_legendre_all(n, x)
            dp = n * (x * P[n] - P[n - 1]) / (x * x - 1)
            dx = P[n] / dp
            x -= dx
            if abs(dx) < mp.mpf(10) ** (-mp.mp.dps + 3):
                break
        P = _mp_legendre_all(n, x)
        dp = n * (x * P[n] - P[n - 1]) / (x * x - 1)
        xs.append(x)
        ws.append(2 / ((1 - x * x) * dp * dp))
    return xs, ws


@functools.lru_cache(maxsize=None)
def _mp_patterson(ext):
    """Gauss-Patterson nodes/weights on [-1,1] at 60 digits: Kronrod-Patterson extensions of the
    1-point Gauss rule; each extension's m+1 new nodes are the zeros of the polynomial of degree
    m+1 orthogonal to all polynomials of degree <= m against prod(x - old nodes) (mpmath findroot
    between consecutive old nodes); weights from the exact integrals of the Lagrange basis."""
    with mp.workdps(60):
        t = [mp.mpf(0)]
        for _ in range(ext):
            m = len(t)
            xs, ws = _mp_gauss(2 * m + 2)
            pm = [mp.fprod([x - a for a in t]) for x in xs]
            Ps = [_mp_legendre_all(m + 1, x) for x in xs]
            # G has the parity of m+1 (even), prod(x - old) that of m (odd): only odd test
            # polynomials P_i give nontrivial conditions, on the even coefficients of G
            idx = [j for j in range(m + 1) if j % 2 == 0]
            rows = [i for i in range(m + 1) if i % 2 == 1]
            A = mp.matrix(len(rows), len(idx))
            b = mp.matrix(len(rows), 1)
            for r, i in enumerate(rows):
                for c, j in enumerate(idx):
                    A[r, c] = mp.fsum(w * P[i] * P[j] * p for w, P, p in zip(ws, Ps, pm))
                b[r] = -mp.fsum(w * P[i] * P[m + 1] * p for w, P, p in zip(ws, Ps, pm))
            a = mp.lu_solve(A, b)

            def G(x, a=a, m=m, idx=idx):
                P = _mp_legendre_all(m + 1, x)
                return P[m + 1] + mp.fsum(a[c] * P[j] for c, j in enumerate(idx))

            ends = [mp.mpf(-1)] + t + [mp.mpf(1)]
            t = sorted(t + [mp.findroot(G, (lo, hi), solver="anderson")
                            for lo, hi in zip(ends[:-1], ends[1:])])
        n = len(t)
        xs, ws = _mp_gauss(n // 2 + 2)
        w = [mp.fsum(W * mp.fprod([(X - t[i]) / (t[j] - t[i]) for i in range(n) if i != j])
                     for X, W in zip(xs, ws)) for j in range(n)]
        return t, w


def node_count(rule: int, level: int) -> int:
    if rule in (S.RULE_CC, S.RULE_TRAP):
        return 1 if level == 1 else 2 ** (level - 1) + 1
    if rule == S.RULE_GP:
        return 2 ** (gp_extensions(level) + 1) - 1
    return level


def coef(d: int, L: int, e: int) -> int:
    """(-1)^{q-|l|} C(d-1, q-|l|) with q = d+L, |l| = d+e; 0 outside the band."""
    from math import comb
    if e < 0 or e > L or L - e > d - 1:
        return 0
    return (-1) ** (L - e) * comb(d - 1, L - e)


def _factor(kind, ck, wk, x):
    x = mp.mpf(x)
    ck = mp.mpf(ck)
    if kind == S.KIND_EXP:
        return mp.exp(ck * x)
    if kind == S.KIND_OSC:
        return mp.expj(ck * x)
    if kind == S.KIND_PEAK:
        wk = mp.mpf(wk)
        return 1 / (1 / (ck * ck) + (x - wk) ** 2)
    if kind == S.KIND_GAUSS:
        wk = mp.mpf(wk)
        return mp.exp(-(ck * ck) * (x - wk) ** 2)
    raise ValueError(kind)


def dp_value(p: S.Problem, form: str = "combination", rules=None):
    """Exact A(d+L, d) f (50 digits) for the product-form kinds, from float64 rule tables.

    form = "combination": Eq 2.6 coefficients;  form = "delta": sum_{|i|<=q} prod Delta^{i_k}
    (reading R6 of Eq 2.9), which must agree to all digits.
    """
    rules = rules or mp_rule
    d, L = p.d, p.L
    with mp.workdps(DPS):
        tabs = {l: rules(p.rule, l) for l in range(1, L + 2)}
        poly_total = [mp.mpf(1)] + [mp.mpf(0)] * L
        for k in range(d):
            wk = None if p.w is None else p.w[k]
            J = []
            for l in range(1, L + 2):
                xs, ws = tabs[l]
                J.append(mp.fsum(mp.mpf(wj) * _factor(p.kind, p.c[k], wk, xj)
                                 for xj, wj in zip(xs, ws)))
            if form == "delta":
                J = [J[0]] + [J[i] - J[i - 1] for i in range(1, len(J))]
            new = [mp.mpf(0)] * (L + 1)
            for a in range(L + 1):
                if poly_total[a] == 0:
                    continue
                for b in range(L + 1 - a):
                    new[a + b] += poly_total[a] * J[b]
            poly_total = new
        if form == "delta":
            s = mp.fsum(poly_total)
        else:
            s = mp.fsum(coef(d, L, e) * poly_total[e] for e in range(L + 1))
        if p.kind == S.KIND_OSC:
            s = mp.re(mp.expj(2 * mp.pi * mp.mpf(p.u)) * s)
        return s


def closed_form(p: S.Problem):
    """Exact integral over [0,1]^d (BASELINE.json configs' closed forms)."""
    with mp.workdps(DPS):
        if p.kind == S.KIND_EXP:
            r = mp.mpf(1)
            for ck in p.c:
                ck = mp.mpf(ck)
                r *= (mp.exp(ck) - 1) / ck if ck != 0 else 1
            return r
        if p.kind == S.KIND_OSC:
            r = mp.expj(2 * mp.pi * mp.mpf(p.u))
            for ck in p.c:
                ck = mp.mpf(ck)
                r *= (mp.expj(ck) - 1) / (1j * ck)
            return mp.re(r)
        if p.kind == S.KIND_PEAK:
            r = mp.mpf(1)
            for ck, wk in zip(p.c, p.w):
                ck, wk = mp.mpf(ck), mp.mpf(wk)
                r *= ck * (mp.atan(ck * (1 - wk)) + mp.atan(ck * wk))
            return r
        if p.kind == S.KIND_GAUSS:
            r = mp.mpf(1)
            for ck, wk in zip(p.c, p.w):
                ck, wk = mp.mpf(ck), mp.mpf(wk)
                r *= mp.sqrt(mp.pi) / (2 * ck) * (mp.erf(ck * (1 - wk)) + mp.erf(ck * wk))
            return r
        if p.kind == S.KIND_CORNER:
            # d-fold integration of (1 + c.x)^-(d+1): each step int_0^1 (a + c x)^-(n+1) dx =
            # (a^-n - (a + c)^-n) / (n c), so I = sum_{v in {0,1}^d} (-1)^|v| / (1 + c.v) / (d! prod c)
            # (all c_k != 0; exponential in d, cancelling: only for small d at 50 digits)
            import itertools
            d = p.d
            tot = mp.mpf(0)
            for v in itertools.product((0, 1), repeat=d):
                tot += (-1) ** sum(v) / (1 + mp.fsum(mp.mpf(ci) for ci, vi in zip(p.c, v) if vi))
            return tot / (mp.factorial(d) * mp.fprod([mp.mpf(ci) for ci in p.c]))
    raise ValueError(p.kind)


def point_count(rule: int, d: int, L: int) -> list[int]:
    """#points per excess class e: [z^e] (sum_l n_l z^{l-1})^d."""
    g = [node_count(rule, l) for l in range(1, L + 2)]
    poly = [1] + [0] * L
    for _ in range(d):
        new = [0] * (L + 1)
        for a in range(L + 1):
            if poly[a]:
                for b in range(L + 1 - a):
                    new[a + b] += poly[a] * g[b]
        poly = new
    return poly


def n_points(rule: int, d: int, L: int) -> int:
    """n_d^q with q = d + L: points in the band e >= L - d + 1."""
    pc = point_count(rule, d, L)
    return sum(pc[e] for e in range(max(0, L - d + 1), L + 1))
