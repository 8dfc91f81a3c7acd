"""The double-double constants of the library's table-driven exp / sin / cos (csrc/dd.cuh) against
60-digit mpmath values, on the CPU: every (hi, lo) pair is the correctly split value of its
definition (|hi + lo - x| <= 2^-104 |x|, hi = fl(x)), so a mistyped or shifted table entry fails here
before any GPU run.  (The device functions themselves are pinned through the factor tables by
tests/test_gpu_parity.py::test_factor_table_matches_mpmath.)"""
import os
import re

import mpmath as mp
import pytest

mp.mp.dps = 60
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
SRC = open(os.path.join(ROOT, "paper_2210_14313_b200", "csrc", "dd.cuh")).read()


def table(name):
    m = re.search(name + r"\[(\d+)\]\[2\] = \{(.*?)\n\};", SRC, re.S)
    assert m, name
    pairs = re.findall(r"\{([-+0-9.e]+), ([-+0-9.e]+)\}", m.group(2))
    assert len(pairs) == int(m.group(1))
    return [(float(a), float(b)) for a, b in pairs]


DEFS = {
    "DD_EXP_C": lambda k: 1 / mp.factorial(k + 1),
    "DD_EXP_TAB": lambda i: mp.exp(mp.mpf(i - 23) / 64),
    "DD_SIN_C": lambda k: (-1) ** k / mp.factorial(2 * k + 1),
    "DD_COS_C": lambda k: (-1) ** k / mp.factorial(2 * k),
    "DD_SINPI64": lambda j: mp.sin(j * mp.pi / 64),
    "DD_COSPI64": lambda j: mp.cos(j * mp.pi / 64),
}


@pytest.mark.parametrize("name", sorted(DEFS))
def test_dd_table_entries(name):
    for i, (hi, lo) in enumerate(table(name)):
        x = DEFS[name](i)
        if x == 0:
            assert hi == 0.0 and lo == 0.0
            continue
        assert hi == float(x), (name, i)
        assert abs(mp.mpf(hi) + mp.mpf(lo) - x) <= mp.mpf(2) ** -104 * abs(x), (name, i)


def test_dd_scalar_constants():
    def const(n):
        return float(re.search(r"#define " + n + r" ([-+0-9.e]+)", SRC).group(1))
    p = mp.pi / 64
    parts = [const("DD_PI64_0"), const("DD_PI64_1"), const("DD_PI64_2")]
    assert abs(sum(mp.mpf(v) for v in parts) - p) <= mp.mpf(2) ** -150 * p
    assert const("DD_64_PI") == float(64 / mp.pi)
    assert const("DD_INV_LN2") == float(1 / mp.log(2))
    ln2 = mp.mpf(const("DD_LN2_HI")) + mp.mpf(const("DD_LN2_LO"))
    assert abs(ln2 - mp.log(2)) <= mp.mpf(2) ** -104
