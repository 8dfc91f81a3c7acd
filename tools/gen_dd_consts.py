"""Generate the double-double constants of the table-driven dd exp / sin / cos (csrc/dd.cuh).

    python tools/gen_dd_consts.py > /tmp/dd_consts.h

Every constant is a 60-digit mpmath value split into hi = fl(x), lo = fl(x - hi).  Not part of the
product path: the output is pasted into dd.cuh once (the values are checked there by
tests/test_gpu_parity.py::test_factor_table_matches_mpmath through the factor tables).
"""
import mpmath as mp

mp.mp.dps = 60


def dd(x):
    hi = float(x)
    lo = float(x - mp.mpf(hi))
    return f"{{{hi!r}, {lo!r}}}"


def arr(name, vals, comment):
    print(f"// {comment}")
    print(f"__device__ __constant__ double {name}[{len(vals)}][2] = {{")
    print(",\n".join("    " + dd(v) for v in vals))
    print("};")


arr("DD_EXP_C", [1 / mp.factorial(k + 1) for k in range(12)], "1/(k+1)!, k = 0..11 (exp(s) - 1 = s sum_k s^k/(k+1)!)")
arr("DD_EXP_TAB", [mp.exp(mp.mpf(j) / 64) for j in range(-23, 24)], "exp(j/64), j = -23..23 (index j + 23)")
arr("DD_SIN_C", [(-1) ** k / mp.factorial(2 * k + 1) for k in range(8)], "(-1)^k/(2k+1)!, k = 0..7")
arr("DD_COS_C", [(-1) ** k / mp.factorial(2 * k) for k in range(8)], "(-1)^k/(2k)!, k = 0..7")
arr("DD_SINPI64", [mp.sin(j * mp.pi / 64) for j in range(17)], "sin(j pi/64), j = 0..16")
arr("DD_COSPI64", [mp.cos(j * mp.pi / 64) for j in range(17)], "cos(j pi/64), j = 0..16")
p = mp.pi / 64
p0 = float(p)
p1 = float(p - mp.mpf(p0))
p2 = float(p - mp.mpf(p0) - mp.mpf(p1))
print(f"#define DD_PI64_0 {p0!r}\n#define DD_PI64_1 {p1!r}\n#define DD_PI64_2 {p2!r}")
print(f"#define DD_64_PI {float(64 / mp.pi)!r}\n#define DD_INV_LN2 {float(1 / mp.log(2))!r}")
