"""Pins for the CPU oracle (oracle/oracle.c), independent of its own code.

Each test pins an oracle function against something other than itself:
SPEC.md worked examples (tests/golden/spec_examples.txt), closed forms,
invariants the paper states, the paper's own Functions executed at small
word sizes (an independent algorithm), Python's big-integer arithmetic (a
library routine), or brute force on tiny inputs.  No GPU needed.
"""
import os
import random

import numpy as np
import pytest

from gen import config_seed, limbs16, residues

HERE = os.path.dirname(os.path.abspath(__file__))
P30 = 998244353          # 119 * 2^23 + 1, generator 3 (C1, C3)
P32 = 3221225473         # 3 * 2^30 + 1, generator 5 (C2)
PG = (1 << 64) - (1 << 32) + 1   # Goldilocks, generator 7 (C4, C5)
P29 = 469762049          # 7 * 2^26 + 1 (the paper's FFT prime)


# ---------------------------------------------------------------- golden
def _golden():
    rows = []
    with open(os.path.join(HERE, "golden", "spec_examples.txt")) as f:
        for line in f:
            line = line.split("#")[0].strip()
            if not line:
                continue
            lhs, z = line.split("->")
            op, p, m, x, y = lhs.split()
            rows.append((op, int(p, 16), int(m), int(x, 16), int(y, 16), int(z, 16)))
    return rows


@pytest.mark.parametrize("row", _golden())
def test_spec_golden(O, row):
    op, p, m, x, y, z = row
    if op == "add_mod":
        assert O.addmod(x, y, p) == z
    elif op == "mul_mod":
        assert O.mulmod(x, y, p) == z
    elif op == "mont_mul":
        assert int(O.vec_montmul([x], [y], p, m)[0]) == z
    elif op == "shoup_psi":
        assert O.shoup_psi(x, p, m) == z
    elif op == "barrett_reduce":
        bp = O.barrett_params(p, m, 2)
        v, it = O.reduce_barrett_fn6(x, p, bp["s"], bp["t"], bp["q"])
        assert v == z and it <= bp["h"]
    elif op == "mont_reduce":
        mp = O.montgomery_params(p, m)
        assert O.reduce_montgomery_fn13(x, p, m, mp["chi"]) == z
    else:
        raise AssertionError(op)


# ---------------------------------------------------------------- primes
def test_primes_and_adicity(O):
    # P:925 "p = 469762049 = 7 x 2^26 + 1"; BASELINE configs fix the others.
    assert O.is_prime(P29) and O.two_adicity(P29) == 26 and P29 == 7 * 2**26 + 1
    assert O.is_prime(P30) and O.two_adicity(P30) == 23 and P30 == 119 * 2**23 + 1
    assert O.is_prime(P32) and O.two_adicity(P32) == 30 and P32 == 3 * 2**30 + 1
    assert O.is_prime(PG) and O.two_adicity(PG) == 32
    # P:973 three primes
    for q in (998244353, 985661441, 943718401):
        assert O.is_prime(q)
    # composites / small cases, brute-force checked
    for n in range(0, 2000):
        brute = n >= 2 and all(n % d for d in range(2, int(n ** 0.5) + 1))
        assert O.is_prime(n) == brute, n
    assert not O.is_prime(PG - 2) or all(pow(a, PG - 3, PG - 2) == 1 for a in (2, 3))


def test_generators_are_primitive(O):
    # g primitive <=> g^((p-1)/l) != 1 for every prime l | p-1 (Python pow as library routine)
    for p, g, fac in ((P30, 3, (2, 7, 17)), (P32, 5, (2, 3)),
                      (PG, 7, (2, 3, 5, 17, 257, 65537))):
        for l in fac:
            assert O.powmod(g, (p - 1) // l, p) == pow(g, (p - 1) // l, p) != 1


def test_root_exact_order(O):
    # BASELINE: "omega having exact order 2^l"; P:887 primitive n-th root.
    for p, g, kmax in ((P30, 3, 23), (P32, 5, 30), (PG, 7, 32)):
        for k in range(0, kmax + 1):
            w = O.root_of_unity(g, k, p)
            assert O.order_pow2(w, k, p) == 1 << k
            if k >= 1:
                assert O.powmod(w, 1 << (k - 1), p) == p - 1


# ---------------------------------------------------------------- scalars
def test_addsub_closed_forms(O):
    for p in (7, 251, P30, P32, PG):
        for x in (0, 1, 2, (p - 1) // 2, p - 2, p - 1):
            assert O.addmod(x, 0, p) == x
            assert O.addmod(x, (p - x) % p, p) == 0
            assert O.submod(x, x, p) == 0
            assert O.submod(0, x, p) == (p - x) % p
        assert O.addmod(p - 1, p - 1, p) == p - 2
        assert O.submod(0, 1, p) == p - 1


def _fn1_add_mod(x, y, p, n):
    """Function 1 executed in n-bit unsigned words."""
    M = (1 << n) - 1
    a = (x + y) & M
    if a < x:
        return (a - p) & M
    return (a - p) & M if a >= p else a


def _fn4_add_mod_epu(x, y, p, n):
    """Function 4, m = n, on one n-bit lane."""
    M = (1 << n) - 1
    a = (p - y) & M
    b = max(x, a) == x
    c = 0 if b else p
    return ((x - a) + c) & M


def _fn2_add_mod_1(x, y, p, n):
    """Function 2, m <= n-1."""
    M = (1 << n) - 1
    a = (x + y) & M
    return min(a, (a - p) & M)


def test_add_vs_paper_functions_bruteforce(O):
    # the paper's Functions 1, 2, 4 are independent algorithms for the same
    # definition; all agree with the oracle on every pair, every p < 2^8.
    n = 8
    for p in range(2, 256):
        for x in range(p):
            for y in range(0, p, max(1, p // 37)):
                z = O.addmod(x, y, p)
                assert _fn1_add_mod(x, y, p, n) == z
                assert _fn4_add_mod_epu(x, y, p, n) == z
                if p < 128:
                    assert _fn2_add_mod_1(x, y, p, n) == z


def test_fn3_printed_line3_is_wrong_corrected_is_right(O):
    # DESIGN.md R2: Function 3 line 3 as printed returns b + (b & p);
    # the intended a + (b & p) is what matches the definition.
    n, M = 8, 255
    wrong = 0
    for p in range(3, 128, 2):
        for x in range(p):
            for y in range(p):
                a = (x + y - p) & M
                b = M if (a >= 128) else 0          # _mm_cmpgt_epi64(0, a): a < 0 as signed
                fixed = (a + (b & p)) & M
                printed = (b + (b & p)) & M
                assert fixed == O.addmod(x, y, p)
                wrong += printed != fixed
    assert wrong > 0


def test_mulmod_closed_forms(O):
    for p in (7, 251, P30, P32, PG):
        for x in (0, 1, 2, p - 2, p - 1, (p - 1) // 2):
            assert O.mulmod(x, 0, p) == 0
            assert O.mulmod(x, 1, p) == x
        assert O.mulmod(p - 1, p - 1, p) == 1            # (-1)^2
        assert O.mulmod(p - 1, 2, p) == p - 2             # -2
    # Goldilocks identities: 2^64 = 2^32 - 1, 2^96 = -1
    assert O.powmod(2, 64, PG) == (1 << 32) - 1
    assert O.powmod(2, 96, PG) == PG - 1
    assert O.powmod(2, 192, PG) == 1


def test_mulmod_vs_python_bigint(O):
    rng = random.Random(1)
    for p in (P30, P32, PG, 3, 65537):
        for _ in range(2000):
            x, y = rng.randrange(p), rng.randrange(p)
            assert O.mulmod(x, y, p) == (x * y) % p    # Python big-int arithmetic
        # boundary products near 2^128 for Goldilocks
    for x in (PG - 1, PG - 2, (1 << 63), (1 << 32) - 1, 1 << 32):
        for y in (PG - 1, (1 << 63) + 5, (1 << 32) + 1):
            assert O.mulmod(x, y, PG) == (x * y) % PG


def test_barrett_table3_and_prop1(O):
    # Table 3 columns for n = 8 and n = 10, every admissible p,
    # Function 6 on every a < alpha p (stride) -- Prop. 1: correct, <= h loops.
    for n in (8, 10):
        for profile, mmax in ((2, n - 2), (1, n - 1), (0, n)):
            maxit = 0
            for p in range(3, 1 << mmax):
                bp = O.barrett_params(p, n, profile)
                assert bp["t"] >= bp["r"] and bp["s"] + bp["t"] <= n + bp["r"] - 1
                assert bp["q"] < (1 << n)
                A = (1 << bp["alpha_log2"]) * p
                step = max(1, A // 257)
                for a in list(range(0, A, step)) + [A - 1]:
                    v, it = O.reduce_barrett_fn6(a, p, bp["s"], bp["t"], bp["q"])
                    assert v == a % p
                    assert it <= bp["h"]
                    maxit = max(maxit, it)
            assert maxit >= 1
    with pytest.raises(ValueError):
        O.barrett_params(2, 8, 2)             # MINUS2 invalid at p = 2


def test_barrett_params_c2(O):
    # FULL profile for the C2 prime (m = n = 32): s = r-1 = 31, t = 32, h = 3
    bp = O.barrett_params(P32, 32, 0)
    assert (bp["r"], bp["s"], bp["t"], bp["h"]) == (32, 31, 32, 3)
    assert bp["q"] == (1 << 63) // P32
    bp = O.barrett_params(P30, 32, 2)
    assert (bp["r"], bp["s"], bp["t"], bp["h"]) == (30, 28, 33, 1)


def _fn8(x, y, psi, p, n):
    """Function 8 in n-bit words."""
    c = (x * psi) >> n
    d = x * y - c * p
    return d - p if d >= p else d


def test_shoup_psi_drives_function8(O):
    # Prop. 4: with psi = floor(2^n y / p), Function 8 returns x y rem p.
    for p in (7, 13, 251):
        for y in range(p):
            psi = O.shoup_psi(y, p, 8)
            assert psi < 256
            for x in range(p):
                assert _fn8(x, y, psi, p, 8) == O.mulmod(x, y, p)
    rng = random.Random(2)
    for p in (P30, P32):
        for _ in range(3000):
            x, y = rng.randrange(p), rng.randrange(p)
            psi = O.shoup_psi(y, p, 32)
            assert psi < (1 << 32)
            assert _fn8(x, y, psi, p, 32) == (x * y) % p
    # psi off by one must break Function 8 somewhere (mutation check)
    p, bad = P32, 0
    for _ in range(3000):
        x, y = rng.randrange(p), rng.randrange(1, p)
        bad += _fn8(x, y, O.shoup_psi(y, p, 32) + 1, p, 32) != (x * y) % p
    assert bad > 0


def test_fn9_needs_ceiling(O):
    # DESIGN.md R4: Function 9 with the printed floor psi fails for
    # some m <= n/2 moduli; ceiling(2^n y / p) passes everywhere (Prop. 5).
    n, M = 16, (1 << 16) - 1
    wrong_floor = 0
    for p in range(2, 256):
        x = np.arange(p, dtype=np.int64)[:, None]
        y = np.arange(p, dtype=np.int64)[None, :]
        fl = (y << n) // p
        ce = -((-(y << n)) // p)
        ref = np.array([[O.mulmod(int(a), int(b), p) for b in range(p)] for a in range(p)]) \
            if p < 16 else (x * y) % p
        zf = (x * y - ((x * fl) >> n) * p) & M
        zc = (x * y - ((x * ce) >> n) * p) & M
        assert np.array_equal(zc, ref)
        wrong_floor += int((zf != ref).sum())
    assert wrong_floor > 0


def test_montgomery_params_and_fn13(O):
    # rho 2^m - chi p = 1, 0 < chi < 2^m, 0 < rho < p; S:126-128 examples.
    assert O.montgomery_params(7, 8)["rho"] == 2 and O.montgomery_params(7, 8)["chi"] == 73
    assert O.montgomery_params(3, 2)["rho"] == 1 and O.montgomery_params(3, 2)["chi"] == 1
    with pytest.raises(ValueError):
        O.montgomery_params(8, 8)
    for p, m in ((P30, 32), (P32, 32), (65537, 32), (P29, 30), (7, 8), (251, 8)):
        mp = O.montgomery_params(p, m)
        assert mp["rho"] * (1 << m) - mp["chi"] * p == 1
        assert 0 < mp["chi"] < (1 << m) and 0 < mp["rho"] < p
        assert mp["r2"] == pow(2, 2 * m, p)
    # Function 13 vs Python bigint: REDC(a) = a rho mod p for a < 2^m p
    rng = random.Random(3)
    for p, m in ((P30, 32), (P32, 32), (251, 8)):
        mp = O.montgomery_params(p, m)
        for _ in range(2000):
            a = rng.randrange((1 << m) * p)
            assert O.reduce_montgomery_fn13(a, p, m, mp["chi"]) == a * mp["rho"] % p


def test_montgomery_roundtrip(O):
    # S:184 from_mont(to_mont(x)) = x; mont_mul(to_mont x, to_mont y) = to_mont(x y)
    for p in (7, 251, P30, P32):
        xs = np.array(sorted({0, 1, 2, p - 2, p - 1, p // 3}), dtype=np.uint64)
        xt = O.vec_to_mont(xs, p, 32)
        back = O.vec_montmul(xt, np.ones_like(xt), p, 32)
        assert np.array_equal(back, xs)
        ys = xs[::-1].copy()
        lhs = O.vec_montmul(xt, O.vec_to_mont(ys, p, 32), p, 32)
        rhs = O.vec_to_mont(O.vec_mulmod(xs, ys, p), p, 32)
        assert np.array_equal(lhs, rhs)


# ---------------------------------------------------------------- NTT
def test_bitrev(O):
    assert O.bitrev(0, 5) == 0 and O.bitrev(1, 3) == 4 and O.bitrev(3, 4) == 12
    for k in range(0, 9):
        perm = [O.bitrev(i, k) for i in range(1 << k)]
        assert sorted(perm) == list(range(1 << k))
        assert all(O.bitrev(perm[i], k) == i for i in range(1 << k))


def test_dft_spec_examples(O):
    # S:327 p = 5, w = 2, a = (1,2,3,4) -> (0,4,3,2); S:336 BITREV -> (0,3,4,2)
    assert list(O.dft([1, 2, 3, 4], 2, 5)) == [0, 4, 3, 2]
    assert list(O.to_bitrev(O.dft([1, 2, 3, 4], 2, 5))) == [0, 3, 4, 2]
    assert list(O.dft([3, 0, 0, 0], 2, 5)) == [3, 3, 3, 3]
    assert list(O.dft([0, 0, 0, 0], 2, 5)) == [0, 0, 0, 0]


@pytest.mark.parametrize("p,g", [(P30, 3), (P32, 5), (PG, 7), (17, 3), (97, 5)])
def test_dft_closed_forms(O, p, g):
    for k in range(0, 7):
        n = 1 << k
        if k > O.two_adicity(p):
            continue
        w = O.root_of_unity(g, k, p)
        for kk in (0, 1, n - 1):
            d = np.zeros(n, dtype=np.uint64); d[kk % n] = 1
            out = O.dft(d, w, p)               # NTT(delta_k)_i = w^(i k)
            assert [int(v) for v in out] == [pow(w, i * (kk % n), p) for i in range(n)]
        c = 12345 % p
        out = O.dft(np.full(n, c, dtype=np.uint64), w, p)  # NTT(const c) = (n c, 0, ..)
        assert int(out[0]) == n * c % p and not out[1:].any()


def test_ntt_equals_dft_all_sizes(O):
    # textbook radix-2 == definition for every n <= 2^12
    for p, g in ((P30, 3), (PG, 7), (P32, 5)):
        for k in range(0, 13):
            a = residues(config_seed(9), k, 1 << k, p).astype(np.uint64)
            w = O.root_of_unity(g, k, p)
            assert np.array_equal(O.ntt(a, w, p), O.dft(a, w, p)), (p, k)
            assert np.array_equal(O.intt(O.ntt(a, w, p), w, p), a)


def test_ntt_linearity_and_roundtrip_large(O):
    p, g, k = P30, 3, 16
    w = O.root_of_unity(g, k, p)
    a = residues(7, 1, 1 << k, p).astype(np.uint64)
    b = residues(7, 2, 1 << k, p).astype(np.uint64)
    s = O.vec_addmod(a, b, p)
    assert np.array_equal(O.ntt(s, w, p), O.vec_addmod(O.ntt(a, w, p), O.ntt(b, w, p), p))
    assert np.array_equal(O.intt(O.ntt(a, w, p), w, p), a)
    for i in (0, 1, 12345, (1 << k) - 1):
        assert O.dft_point(a, w, i, p) == int(O.ntt(a, w, p)[i])


@pytest.mark.parametrize("k,k1", [(3, 1), (4, 2), (5, 3), (5, 2), (8, 4), (9, 3), (10, 5)])
def test_algorithm1_is_bitrev_dft(O, k, k1):
    # Proposition 15: Algorithm 1 (l = n) returns A(w^{[i]_k}) at position i.
    for p, g in ((P30, 3), (PG, 7)):
        a = residues(11, k, 1 << k, p).astype(np.uint64)
        w = O.root_of_unity(g, k, p)
        assert np.array_equal(O.algorithm1(a, k1, w, p), O.to_bitrev(O.dft(a, w, p)))


# ---------------------------------------------------------------- products
def test_poly_mul_closed_forms(O):
    assert list(O.poly_mul_schoolbook([1, 1], [1, 1], 7)) == [1, 2, 1]
    assert list(O.poly_mul_ntt([1, 1], [1, 1], P29, 3)) == [1, 2, 1]
    a = residues(1, 1, 37, P30).astype(np.uint64)
    assert np.array_equal(O.poly_mul_schoolbook(a, [1], P30), a)
    assert list(O.poly_mul_schoolbook([5], [6], 7)) == [2]
    # exact integer convolution (numpy object ints) reduced mod p
    b = residues(1, 2, 23, P30).astype(np.uint64)
    exact = np.convolve(a.astype(object), b.astype(object)) % P30
    assert [int(v) for v in O.poly_mul_schoolbook(a, b, P30)] == [int(v) for v in exact]


def test_poly_mul_ntt_vs_schoolbook(O):
    rng = random.Random(5)
    for p, g in ((P30, 3), (P29, 3), (PG, 7), (P32, 5)):
        for _ in range(12):
            la, lb = rng.randrange(1, 300), rng.randrange(1, 300)
            a = residues(rng.randrange(1 << 30), 1, la, p).astype(np.uint64)
            b = residues(rng.randrange(1 << 30), 2, lb, p).astype(np.uint64)
            c1 = O.poly_mul_schoolbook(a, b, p)
            assert np.array_equal(c1, O.poly_mul_ntt(a, b, p, g))
            assert np.array_equal(c1, O.poly_mul_schoolbook(b, a, p))        # commutativity
            r = rng.randrange(p)
            assert O.poly_eval(c1, r, p) == O.mulmod(O.poly_eval(a, r, p), O.poly_eval(b, r, p), p)


def test_poly_eval_horner(O):
    assert O.poly_eval([1, 2, 3], 10, 1000003) == 321
    assert O.poly_eval([], 5, 7) == 0


def _to_int(limbs):
    return sum(int(v) << (16 * i) for i, v in enumerate(limbs))


def test_int_mul_closed_forms(O):
    # S:501 (2^32 - 1)^2 = 0xFFFFFFFE00000001
    a = [0xFFFF, 0xFFFF]
    c = O.int_mul_schoolbook_u16(a, a)
    assert _to_int(c) == 0xFFFFFFFE00000001
    assert np.array_equal(c, O.int_mul_ntt_u16(a, a))
    # (2^(16N) - 1)^2 limbs = [1, 0 x (N-1), 0xFFFE, 0xFFFF x (N-1)]
    for N in (1, 2, 5, 64, 1000):
        a = np.full(N, 0xFFFF, dtype=np.uint16)
        expect = [1] + [0] * (N - 1) + [0xFFFE] + [0xFFFF] * (N - 1)
        assert list(O.int_mul_ntt_u16(a, a)) == expect
        assert list(O.int_mul_schoolbook_u16(a, a)) == expect
    x = limbs16(3, 1, 50)
    assert not O.int_mul_schoolbook_u16(x, np.zeros(3, np.uint16)).any()      # a 0 = 0
    one = np.zeros(4, np.uint16); one[0] = 1
    assert np.array_equal(O.int_mul_schoolbook_u16(x, one)[:50], x)          # a 1 = a


def test_int_mul_vs_python_bigint(O):
    rng = random.Random(6)
    for _ in range(20):
        na, nb = rng.randrange(1, 400), rng.randrange(1, 400)
        a, b = limbs16(rng.randrange(1 << 30), 1, na), limbs16(rng.randrange(1 << 30), 2, nb)
        c = O.int_mul_schoolbook_u16(a, b)
        assert _to_int(c) == _to_int(a) * _to_int(b)          # Python big ints (library)
        assert np.array_equal(c, O.int_mul_ntt_u16(a, b))
        q = (1 << 61) - 1
        assert O.limbs_mod(c, q) == (_to_int(a) % q) * (_to_int(b) % q) % q


def test_carry_u16(O):
    rng = random.Random(7)
    coef = [rng.randrange(1 << 56) for _ in range(100)]
    out = O.carry_u16(np.array(coef, dtype=np.uint64), 104)
    assert _to_int(out) == sum(c << (16 * i) for i, c in enumerate(coef))


# ------------------------------------------------------------------ polynomial matrix product
def test_poly_matmul_naive_pins(O):
    p = 469762049                       # Table 15's prime
    rng = np.random.default_rng(15)
    # degree 0: the ordinary matrix product over Z/pZ (numpy object integers)
    A = rng.integers(0, p, size=(3, 4, 1), dtype=np.uint64)
    B = rng.integers(0, p, size=(4, 2, 1), dtype=np.uint64)
    ref = (A[:, :, 0].astype(object) @ B[:, :, 0].astype(object)) % p
    assert np.array_equal(O.poly_matmul_naive(A, B, p)[:, :, 0].astype(object), ref)
    # identity polynomial matrix x B = B (SPEC poly_mat_mul example)
    I = np.zeros((3, 3, 1), dtype=np.uint64)
    for i in range(3):
        I[i, i, 0] = 1
    B = rng.integers(0, p, size=(3, 3, 8), dtype=np.uint64)
    assert np.array_equal(O.poly_matmul_naive(I, B, p), B)
    # entries against Python polynomial arithmetic (x-adic evaluation at 2^64)
    A = rng.integers(0, p, size=(2, 3, 5), dtype=np.uint64)
    B = rng.integers(0, p, size=(3, 2, 4), dtype=np.uint64)
    C = O.poly_matmul_naive(A, B, p)
    for i in range(2):
        for j in range(2):
            coef = [0] * 8
            for l in range(3):
                for u in range(5):
                    for v in range(4):
                        coef[u + v] += int(A[i, l, u]) * int(B[l, j, v])
            assert [int(c) for c in C[i, j]] == [c % p for c in coef]
    # associativity (SPEC property)
    X = rng.integers(0, p, size=(2, 2, 3), dtype=np.uint64)
    Y = rng.integers(0, p, size=(2, 2, 2), dtype=np.uint64)
    Z = rng.integers(0, p, size=(2, 2, 2), dtype=np.uint64)
    assert np.array_equal(O.poly_matmul_naive(O.poly_matmul_naive(X, Y, p), Z, p),
                          O.poly_matmul_naive(X, O.poly_matmul_naive(Y, Z, p), p))


# ---------------------------------------------------------------- order_pow2: negative pins
def test_order_pow2_negatives(O):
    # or_order_pow2 must return the exact order, not just 2^k: w^2 has order
    # 2^(k-1), w^(2^j) order 2^(k-j), -1 order 2, 1 order 1; w has no order
    # dividing 2^(k-1) (w^(2^(k-1)) = -1), and a generator of (Z/pZ)^* (order
    # p - 1, which 2^k does not reach) has none dividing 2^k.  Python pow is
    # the library check of each claim.
    for p, g, kmax in ((P30, 3, 23), (P32, 5, 30), (PG, 7, 32), (P29, 3, 26)):
        for k in (1, 2, 5, kmax - 1, kmax):
            w = O.root_of_unity(g, k, p)
            for j in range(0, k + 1):
                wj = O.powmod(w, 1 << j, p)
                assert O.order_pow2(wj, k, p) == 1 << (k - j), (p, k, j)
            if k >= 1:
                assert pow(w, 1 << (k - 1), p) == p - 1
                assert O.order_pow2(w, k - 1, p) == 0, (p, k)     # order 2^k does not divide 2^(k-1)
            assert O.order_pow2(g, k, p) == 0                     # generator: order p - 1
        assert O.order_pow2(1, 0, p) == 1
        assert O.order_pow2(p - 1, 1, p) == 2
        assert O.order_pow2(p - 1, 0, p) == 0
    # a non-root whose order is odd (> 1): 3^(2^23 * 119... ) -- take g^(2^l) with l the 2-adicity
    for p, g in ((P30, 3), (PG, 7)):
        l = O.two_adicity(p)
        odd = O.powmod(g, 1 << l, p)                              # order (p-1)/2^l, odd and > 1
        assert odd != 1 and O.order_pow2(odd, l, p) == 0


# ---------------------------------------------------------------- definition pins
def _def_pins():
    rows = []
    with open(os.path.join(HERE, "golden", "definition_pins.txt")) as f:
        for line in f:
            line = line.split("#")[0].strip()
            if not line:
                continue
            lhs, rhs = line.split("->")
            p, w, a = lhs.split()
            rows.append((int(p), int(w), [int(x) for x in a.split(",")], [int(x) for x in rhs.split(",")]))
    return rows


@pytest.mark.parametrize("row", _def_pins())
def test_definition_pins(O, row):
    # P:889 FFT_w(a) on SURVEY App. A's (and SPEC S:327's) worked values: the
    # O(n^2) definition, the textbook radix-2 NTT, the BITREV order,
    # Algorithm 1 and the inverse all reproduce them
    p, w, a, ahat = row
    n = len(a)
    k = n.bit_length() - 1
    assert [sum(pow(w, i * j, p) * a[j] for j in range(n)) % p for i in range(n)] == ahat   # library re-derivation
    assert O.order_pow2(w, k, p) == n
    av = np.array(a, dtype=np.uint64)
    assert [int(v) for v in O.dft(av, w, p)] == ahat
    assert [int(v) for v in O.ntt(av, w, p)] == ahat
    bit = [ahat[O.bitrev(i, k)] for i in range(n)]
    assert [int(v) for v in O.to_bitrev(np.array(ahat, dtype=np.uint64))] == bit
    for k1 in range(1, k):
        assert [int(v) for v in O.algorithm1(av, k1, w, p)] == bit
    assert [int(v) for v in O.intt(np.array(ahat, dtype=np.uint64), w, p)] == a
