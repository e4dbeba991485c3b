"""Exact emulation of a binary floating-point type with an l-bit trailing
significand field (paper §3.1: "l represents the size of the mantissa
of F minus one") under the four IEEE-754 rounding modes, for brute-force pins
of Functions 14-16 at small l.

Values are integers scaled by 2^-S (every quantity the functions form is a
multiple of 2^-S for the small l, p used here); each operation is computed
exactly with Python integers and rounded once to l + 1 significant bits, as
IEEE-754 prescribes for *, +, -, fma and /.  Exponent range is unbounded (no
overflow / subnormals: the functions never approach them).  Test
infrastructure only: the CUDA path and the oracle share nothing with it.
"""
from __future__ import annotations

S = 96                       # fixed scale: value = N / 2^S
ONE = 1 << S
RN, RU, RD, RZ = "rn", "ru", "rd", "rz"
MODES = (RN, RU, RD, RZ)


def _round_int_div(num: int, den: int, mode: str) -> int:
    """round(num / den) to an integer in `mode` (den > 0)."""
    q, r = divmod(num, den)          # floor division: num = q den + r, 0 <= r < den
    if r == 0:
        return q
    if mode == RD:
        return q
    if mode == RU:
        return q + 1
    if mode == RZ:
        return q if num >= 0 else q + 1
    # nearest, ties to even
    if 2 * r > den or (2 * r == den and (q & 1)):
        return q + 1
    return q


def rnd_rational(num: int, den: int, ell: int, mode: str) -> int:
    """The F value nearest (in `mode`) to num / den, as an integer at scale S."""
    if num == 0:
        return 0
    if den < 0:
        num, den = -num, -den
    a = abs(num)
    # exponent E with 2^E <= a / den < 2^(E+1)
    E = a.bit_length() - den.bit_length()
    if (a << max(0, -E)) < (den << max(0, E)):
        E -= 1
    # ulp = 2^(E - ell); significand M = round(num / den / ulp)
    sh = E - ell
    if sh >= 0:
        M = _round_int_div(num, den << sh, mode)
    else:
        M = _round_int_div(num << -sh, den, mode)
    # value = M 2^sh (M may have carried to 2^(ell+1): still exact)
    t = sh + S
    assert t >= 0, "value below the emulation scale"
    return M << t


def rnd(N: int, ell: int, mode: str) -> int:
    """Round an exact scaled value N / 2^S to F."""
    return rnd_rational(N, ONE, ell, mode)


def from_int(x: int) -> int:
    return x << S


def to_int(N: int) -> int:
    assert N % ONE == 0, "not an integer"
    return N // ONE


def mul(x: int, y: int, ell: int, mode: str) -> int:
    return rnd_rational(x * y, ONE * ONE, ell, mode)


def fma(x: int, y: int, z: int, ell: int, mode: str) -> int:
    return rnd_rational(x * y + z * ONE, ONE * ONE, ell, mode)


def add(x: int, y: int, ell: int, mode: str) -> int:
    return rnd(x + y, ell, mode)


def sub(x: int, y: int, ell: int, mode: str) -> int:
    return rnd(x - y, ell, mode)


def recip(p: int, ell: int, mode: str) -> int:
    """1.0 / (F) p in `mode` (P:574's u; with RU it is u-bar)."""
    return rnd_rational(1, p, ell, mode)


def floor_(x: int) -> int:
    return (x // ONE) * ONE      # C99 floor: exact in F


# ---------------------------------------------------------------- the paper's functions
def fn14(a: int, p: int, ell: int, mode: str, ubar: bool = False, drop_line4: bool = False) -> int:
    """Function 14 on the integer a, in rounding mode `mode`;
    u = 1/p rounded in `mode` (or u-bar = rounded up).  Returns the integer
    result (lines 4/5 included unless dropped)."""
    A, P = from_int(a), from_int(p)
    u = recip(p, ell, RU if ubar else mode)
    b = mul(A, u, ell, mode)                 # 1. F b = a * u
    c = floor_(b)                            # 2. F c = floor(b)
    d = sub(A, mul(c, P, ell, mode), ell, mode)   # 3. F d = a - c * p
    if not drop_line4 and d >= P:            # 4.
        return to_int(sub(d, P, ell, mode))
    if d < 0:                                # 5.
        return to_int(add(d, P, ell, mode))
    return to_int(d)                         # 6.


def fn15(a: int, p: int, ell: int, mode: str) -> int:
    """Function 15: b = a * u-bar, c = floor(b), a - c p, no
    correction; the hypothesis is mode = RU (Remark 12 drops it for p not
    dividing a)."""
    A, P = from_int(a), from_int(p)
    ub = recip(p, ell, RU)
    b = mul(A, ub, ell, mode)
    c = floor_(b)
    return to_int(sub(A, mul(c, P, ell, mode), ell, mode))


def fn16(a1: int, a2: int, p: int, ell: int, mode: str, ubar: bool = False, drop_line7: bool = False) -> int:
    """Function 16 in rounding mode `mode`."""
    X, Y, P = from_int(a1), from_int(a2), from_int(p)
    u = recip(p, ell, RU if ubar else mode)
    h = mul(X, Y, ell, mode)                 # 1. h = a1 * a2
    l = fma(X, Y, -h, ell, mode)             # 2. l = fma(a1, a2, -h)
    b = mul(h, u, ell, mode)                 # 3. b = h * u
    c = floor_(b)                            # 4. c = floor(b)
    d = fma(-c, P, h, ell, mode)             # 5. d = fma(-c, p, h)
    e = add(d, l, ell, mode)                 # 6. e = d + l
    if not drop_line7 and e >= P:            # 7.
        return to_int(sub(e, P, ell, mode))
    if e < 0:                                # 8.
        return to_int(add(e, P, ell, mode))
    return to_int(e)                         # 9.
