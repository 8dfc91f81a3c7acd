"""Seeded synthetic inputs for the Smolyak hot path (shared by the oracle tests and the CUDA path).

This module holds NO arithmetic of the method: it only names the BASELINE.json workloads and draws
their random integrand parameters.  Both the oracle (``oracle/``) and the CUDA library receive the
same float64 arrays produced here.

Draw convention (SURVEY.md §8c reading G9, DESIGN.md "Readings" R9):
``numpy.random.default_rng(seed)``; ``uniform(lo, hi, d)`` for c, then ``uniform(0, 1, d)`` for w
(if the kind has shifts), then ``uniform(0, 1)`` for u (if the kind has a phase); then, for the
configs that fix Σc, ``c <- c * (S / c.sum())`` in float64.

Workloads: BASELINE.json ``configs[0..4]`` (domain [0,1]^d, q = d + L, Eq 2.6) plus the
paper's own Table 5.6-5.8 integrands mapped to [0,1]^d (SURVEY.md §8c pin P6).
"""
from __future__ import annotations

import math
from dataclasses import dataclass, field

import numpy as np

# Rule ids follow the paper's r parameter: 2 = Clenshaw-Curtis, 4 = Gauss-Legendre.
RULE_TRAP = 1   # trapezoidal (Eq 2.10)
RULE_CC = 2
RULE_GP = 3     # Gauss-Patterson, delayed sequence
RULE_GL = 4
# Integrand kinds (BASELINE.json configs; Genz families).
KIND_EXP = 0      # exp(sum c_k x_k)
KIND_OSC = 1      # cos(2 pi u + sum c_k x_k)
KIND_PEAK = 2     # prod (c_k^-2 + (x_k - w_k)^2)^-1
KIND_GAUSS = 3    # exp(-sum c_k^2 (x_k - w_k)^2)
KIND_CORNER = 4   # (1 + sum c_k x_k)^-(d+1)  (Genz corner peak; not separable: s-form dd path)

KIND_NAMES = {KIND_EXP: "exp", KIND_OSC: "osc", KIND_PEAK: "peak", KIND_GAUSS: "gauss",
              KIND_CORNER: "corner_peak"}
RULE_NAMES = {RULE_TRAP: "trapezoidal", RULE_CC: "clenshaw_curtis", RULE_GP: "gauss_patterson",
              RULE_GL: "gauss_legendre"}


@dataclass
class Problem:
    name: str
    d: int
    L: int                 # level budget above the all-ones multi-index: q = d + L
    rule: int
    kind: int
    c: np.ndarray
    w: np.ndarray | None = None
    u: float = 0.0
    note: str = ""
    meta: dict = field(default_factory=dict)

    @property
    def q(self) -> int:
        return self.d + self.L

    def w_or_zeros(self) -> np.ndarray:
        return self.w if self.w is not None else np.zeros(self.d)


def _draw(seed: int, d: int, c_lo: float, c_hi: float, has_w: bool, has_u: bool,
          c_sum: float | None):
    rng = np.random.default_rng(seed)
    c = rng.uniform(c_lo, c_hi, d)
    w = rng.uniform(0.0, 1.0, d) if has_w else None
    u = float(rng.uniform(0.0, 1.0)) if has_u else 0.0
    if c_sum is not None:
        c = c * (c_sum / c.sum())
    return np.ascontiguousarray(c, dtype=np.float64), (
        None if w is None else np.ascontiguousarray(w, dtype=np.float64)), u


def baseline_config(i: int) -> Problem:
    """BASELINE.json configs[i-1] for i = 1..5."""
    if i == 1:
        c, w, u = _draw(0, 4, 0.0, 1.0, False, False, None)
        return Problem("c1", 4, 4, RULE_CC, KIND_EXP, c, w, u)
    if i == 2:
        c, w, u = _draw(1, 10, 0.0, 1.0, False, True, 9.0)
        return Problem("c2", 10, 6, RULE_CC, KIND_OSC, c, w, u)
    if i == 3:
        c, w, u = _draw(2, 100, 0.5, 1.5, True, False, None)
        return Problem("c3", 100, 4, RULE_GL, KIND_PEAK, c, w, u)
    if i == 4:
        c, w, u = _draw(3, 1000, 0.0, 0.5, True, False, None)
        return Problem("c4", 1000, 3, RULE_CC, KIND_GAUSS, c, w, u)
    if i == 5:
        c, w, u = _draw(4, 300, 0.0, 1.0, False, True, 30.0)
        return Problem("c5", 300, 4, RULE_CC, KIND_OSC, c, w, u)
    raise ValueError(f"no BASELINE config {i}")


def paper_table_problem(table: str, d: int, N: int) -> Problem:
    """Tables 5.6/5.7/5.8 integrands (PAPER.md:619 Test 8) mapped from [-1,1]^d to [0,1]^d.

    x = 2y - 1 (reading R2); relative errors are invariant under the constant factors this drops:
      f  = exp(sum (-1)^{i+1} x_i)           -> exp kind, c_k = 2(-1)^{k+1}
      f^ = cos(2 pi + sum x_i)               -> osc kind, c_k = 2, 2 pi u = 2 pi - d
      f~ = prod 1/(0.9^2 + (x_i - 0.6)^2)    -> peak kind, c_k = 1/0.45, w_k = 0.8
    The paper's p(N) is the maximal 1-D GL level, i.e. L = N - 1.
    """
    L = N - 1
    k = np.arange(d)
    if table == "5.6":
        c = 2.0 * np.where(k % 2 == 0, 1.0, -1.0)
        return Problem(f"T5.6_d{d}_N{N}", d, L, RULE_GL, KIND_EXP, c)
    if table == "5.7":
        c = np.full(d, 2.0)
        u = 1.0 - d / (2.0 * math.pi)
        return Problem(f"T5.7_d{d}_N{N}", d, L, RULE_GL, KIND_OSC, c, None, u)
    if table == "5.8":
        c = np.full(d, 1.0 / 0.45)
        w = np.full(d, 0.8)
        return Problem(f"T5.8_d{d}_N{N}", d, L, RULE_GL, KIND_PEAK, c, w)
    raise ValueError(table)


def corner_config(d: int = 100, L: int = 4, rule: int = RULE_CC, seed: int = 5) -> Problem:
    """Extra (non-BASELINE) workload for the non-separable s-form dd path: Genz corner peak
    (1 + sum c_k x_k)^-(d+1), c_k ~ U(0,1) from `seed` rescaled to sum c_k = 1 (reading R9 draw
    order); d = 100, L = 4, Clenshaw-Curtis by default."""
    c, w, u = _draw(seed, d, 0.0, 1.0, False, False, 1.0)
    return Problem(f"cp_d{d}_L{L}", d, L, rule, KIND_CORNER, c, w, u)


def random_problem(seed: int, d: int, L: int, rule: int, kind: int) -> Problem:
    """Small seeded problems for parity sweeps (same draw convention, generic parameter ranges)."""
    c_lo, c_hi = {KIND_EXP: (-1.0, 1.0), KIND_OSC: (0.0, 1.0), KIND_PEAK: (0.5, 1.5),
                  KIND_GAUSS: (0.0, 0.5), KIND_CORNER: (0.0, 1.0)}[kind]
    has_w = kind in (KIND_PEAK, KIND_GAUSS)
    has_u = kind == KIND_OSC
    # corner peak: Genz-style normalisation sum c_k = 1 (f ranges over (2^-(d+1), 1])
    c, w, u = _draw(seed, d, c_lo, c_hi, has_w, has_u, 1.0 if kind == KIND_CORNER else None)
    return Problem(f"rand_s{seed}_d{d}_L{L}_r{rule}_k{kind}", d, L, rule, kind, c, w, u)
