"""Brute-force pins of the paper's numeric reductions (§3) --
Functions 14, 15 and 16 executed step by step in an exact emulation of a
binary float with an l-bit trailing field under the four IEEE-754 rounding
modes (tests/numeric_emul.py), over every input of their stated domains for
small l.  They pin the readings DESIGN.md R16-R18 takes for the CUDA kernels
(csrc/numeric.cu), whose results the GPU tests compare with the oracle's
plain definition (x y) rem p:

* Proposition 10: Function 14 is correct in every rounding mode;
  with u-bar and rounding toward +inf its line 4 can be dropped -- and it
  cannot be dropped with u (negative pin).
* Proposition 11: Function 15 (u-bar, toward +inf, no correction) is
  correct; with u in place of u-bar it is not (negative pin).
* Remark 12: for p prime and a a product of two residues the
  rounding-mode hypothesis can be dropped.
* Proposition 13: Function 16 is correct in every mode; with u-bar
  and toward +inf its line 7 can be dropped -- and not with u (negative pin).
"""
import pytest

import numeric_emul as E


def _primes(lo, hi):
    return [n for n in range(max(lo, 3), hi) if all(n % d for d in range(2, int(n ** 0.5) + 1))]


@pytest.mark.parametrize("ell", [8, 10])
def test_fn14_prop10(ell):
    # every p with m <= l/2 (p < 2^(l/2)), every a < alpha p, alpha = 2^(l/2)
    alpha = 1 << (ell // 2)
    for p in range(3, 1 << (ell // 2)):
        for a in range(alpha * p):
            for mode in E.MODES:
                assert E.fn14(a, p, ell, mode) == a % p, (ell, p, a, mode)
            # second clause: u-bar and rounding toward +inf, line 4 discarded
            assert E.fn14(a, p, ell, E.RU, ubar=True, drop_line4=True) == a % p, (ell, p, a)


def test_fn14_line4_needed_without_ubar():
    # negative pin: with u = 1/p rounded to nearest (or down) and the same mode
    # for the products, dropping line 4 is wrong for some a
    ell, h = 10, 5
    for mode in (E.RN, E.RD):
        bad = [(p, a) for p in range(3, 1 << h) for a in range(p << h)
               if E.fn14(a, p, ell, mode, drop_line4=True) != a % p]
        assert bad, mode


@pytest.mark.parametrize("ell", [9, 11])
def test_fn15_prop11(ell):
    m = (ell - 1) // 2                 # m <= (l - 1)/2, alpha = 2^((l-1)/2)
    alpha = 1 << m
    for p in range(3, 1 << m):
        for a in range(alpha * p):
            assert E.fn15(a, p, ell, E.RU) == a % p, (ell, p, a)


@pytest.mark.parametrize("ell", [9, 11])
def test_fn15_remark12_products(ell):
    # p prime, a = x y with x, y residues: correct in round-to-nearest too
    m = (ell - 1) // 2
    for p in _primes(3, 1 << m):
        for x in range(p):
            for y in range(p):
                assert E.fn15(x * y, p, ell, E.RN) == (x * y) % p, (ell, p, x, y)


def test_fn15_needs_ubar():
    # negative pin: Function 15 with u (1/p rounded down) instead of u-bar, products
    # rounded down, returns p + (a rem p) for some a
    ell, m = 9, 4
    bad = []
    for p in range(3, 1 << m):
        u = E.recip(p, ell, E.RD)
        for a in range(p << m):
            A, P = E.from_int(a), E.from_int(p)
            c = E.floor_(E.mul(A, u, ell, E.RD))
            if E.to_int(E.sub(A, E.mul(c, P, ell, E.RD), ell, E.RD)) != a % p:
                bad.append((p, a))
    assert bad


def test_fn16_prop13():
    # every p < 2^(l-2) (m <= l - 2) and every pair of residues (a1 a2 < p^2 <= alpha p)
    ell = 8
    for p in range(3, 1 << (ell - 2)):
        for a1 in range(p):
            for a2 in range(p):
                r = (a1 * a2) % p
                for mode in E.MODES:
                    assert E.fn16(a1, a2, p, ell, mode) == r, (p, a1, a2, mode)
                assert E.fn16(a1, a2, p, ell, E.RU, ubar=True, drop_line7=True) == r, (p, a1, a2)


def test_fn16_prop13_wider_sampled():
    # l = 10 (m <= 8): primes near the bound, all pairs for a few, boundary rows for the rest
    ell = 10
    for p in (251, 241, 239, 127, 97):
        for a1 in range(p):
            for a2 in (range(p) if p < 130 else (0, 1, 2, p // 2, p - 2, p - 1, a1)):
                r = (a1 * a2) % p
                for mode in E.MODES:
                    assert E.fn16(a1, a2, p, ell, mode) == r
                assert E.fn16(a1, a2, p, ell, E.RU, ubar=True, drop_line7=True) == r


def test_fn16_line7_needed_without_ubar():
    ell = 8
    bad = [(p, a1, a2) for p in range(3, 64) for a1 in range(p) for a2 in range(p)
           if E.fn16(a1, a2, p, ell, E.RN, drop_line7=True) != (a1 * a2) % p]
    assert bad
