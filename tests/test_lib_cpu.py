"""CPU-side checks of the C-ABI library (no GPU): it builds for sm_100a,
loads, exports every symbol include/mmntt.h declares, and its host-side
argument validation returns the documented statuses without touching a GPU."""
import ctypes
import os
import re
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.fixture(scope="module")
def mm():
    import torch  # noqa: F401  (loads libcudart before libmmntt)
    from paper_1407_3383_b200._build import build
    build()
    import paper_1407_3383_b200 as m
    m.lib()
    return m


def _header_functions():
    src = open(os.path.join(ROOT, "include", "mmntt.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(mm_[a-z0-9_]+)\s*\(", src)))


def test_header_symbols_exported(mm):
    names = _header_functions()
    assert len(names) >= 20
    L = mm.lib()
    for n in names:
        assert hasattr(L, n), n
        assert n in mm.EXPORTS, n
    out = subprocess.run(["nm", "-D", "--defined-only", mm._LIB_PATH], capture_output=True, text=True).stdout
    for n in names:
        assert re.search(rf"\bT {n}\b", out), n


def test_sass_is_sm100a(mm):
    out = subprocess.run(["/usr/local/cuda/bin/cuobjdump", "--list-elf", mm._LIB_PATH],
                         capture_output=True, text=True).stdout
    assert "sm_100a" in out


def test_status_codes_host_side(mm):
    L = mm.lib()
    h = ctypes.c_void_p()
    assert L.mm_mod32_create(4, ctypes.byref(h)) == 1          # even -> invalid modulus
    assert L.mm_mod32_create(2, ctypes.byref(h)) == 1
    assert L.mm_mod32_create(91, ctypes.byref(h)) == 1         # 7 * 13 composite
    assert b"prime" in L.mm_last_error()
    # NTT plan argument validation happens before any device work
    P30 = 998244353
    assert L.mm_ntt_plan_create(32, 3221225473, 10, 5, 1, ctypes.byref(h)) == 2   # p >= 2^30: profile
    assert L.mm_ntt_plan_create(32, P30, 24, 3, 1, ctypes.byref(h)) == 3          # 2^24 does not divide p-1
    assert L.mm_ntt_plan_create(32, P30, 10, 2, 1, ctypes.byref(h)) == 4          # 2 is not a 2^10-th root
    assert L.mm_ntt_plan_create(64, P30, 10, 2, 1, ctypes.byref(h)) == 1          # 64-bit: Goldilocks only
    assert L.mm_ntt_plan_create(16, P30, 10, 2, 1, ctypes.byref(h)) == 10
    assert L.mm_ntt_plan_create(32, P30, 10, 3, 0, ctypes.byref(h)) == 10         # batch 0
    assert L.mm_poly_mul(32, P30, 3, None, 1, None, 1, None, 1, None) == 10
    # int_mul coefficient bound: min(na, nb) (2^16-1)^2 must stay below p
    dummy = ctypes.c_void_p(1 << 40)
    dummy2 = ctypes.c_void_p(1 << 41)
    dummy3 = ctypes.c_void_p(1 << 42)
    assert L.mm_int_mul_u16(dummy, 1 << 33, dummy2, 1 << 33, dummy3, None) == 6
    # aliasing is rejected
    assert L.mm_int_mul_u16(dummy, 100, dummy2, 100, dummy, None) == 7


def test_gold_shift_constants():
    # gold.cuh compiles its 64-th-root twiddles as shifts: w_64 = 2^S_FWD for the
    # canonical root 7^((p-1)/n), 2^S_INV for its inverse, and
    # every 8th / 4th root used by its 8- / 4-point kernels is 2^(8S) / 2^(16S)
    # with 2^96 = -1 (Pow2's (NEG, C) split); recomputed here with Python integers
    src = open(os.path.join(ROOT, "paper_1407_3383_b200", "csrc", "gold.cuh")).read()
    s_fwd = int(re.search(r"S_FWD = (\d+);", src).group(1))
    s_inv = int(re.search(r"S_INV = (\d+);", src).group(1))
    p = (1 << 64) - (1 << 32) + 1
    assert pow(7, (p - 1) // 64, p) == pow(2, s_fwd, p)
    assert pow(2, s_fwd + s_inv, p) == 1
    assert pow(2, 96, p) == p - 1 and pow(2, 192, p) == 1 and pow(2, 64, p) == (1 << 32) - 1
    for S in (s_fwd, s_inv):
        for k in range(192):   # Pow2<k>: 2^k = (-1)^NEG * C with C = 2^(k mod 96) reduced
            kr = k % 96
            c = (1 << kr) if kr < 64 else (1 << (kr - 32)) - (1 << (kr - 64))
            assert c < p and (c if k < 96 else (p - c) % p) == pow(2, k, p)
        # the 8-point kernels' roots: w_8 = 2^(8S) has order 8, w_4 = 2^(16S) order 4
        assert pow(2, 8 * S * 4, p) == p - 1 and pow(2, 16 * S * 2, p) == p - 1


def test_modnum_constants_host_side(mm):
    # mm_modnum_create is host-only: u = 1/p to nearest and u-bar = the
    # least float / double >= 1/p, checked with exact rationals
    from fractions import Fraction
    import numpy as np
    L = mm.lib()
    h = ctypes.c_void_p()
    out = (ctypes.c_double * 6)()
    for fbits in (32, 64):
        l = 52 if fbits == 64 else 23
        ftype = np.float64 if fbits == 64 else np.float32
        for p in (3, 7, 2039, 65537, 2097143, 33554393, 67108859, 1125899906842597, 1108307720798209):
            st = L.mm_modnum_create(fbits, p, ctypes.byref(h))
            if p.bit_length() > l - 2:
                assert st == 2                       # MM_E_PROFILE: m > l - 2 (Function 16's bound)
                continue
            assert st == 0
            assert L.mm_modnum_info(h, out) == 0
            u, ub = Fraction(out[1]), Fraction(out[2])
            assert out[1] == float(ftype(1) / ftype(p))          # nearest
            assert ub >= Fraction(1, p)
            below = Fraction(float(np.nextafter(ftype(out[2]), ftype(0))))
            assert below < Fraction(1, p)                          # least such value
            assert (out[3], out[4], out[5]) == (l, p.bit_length(), fbits)
            L.mm_modnum_destroy(h)
    assert L.mm_modnum_create(64, 4, ctypes.byref(h)) == 1         # even
    assert L.mm_modnum_create(16, 7, ctypes.byref(h)) == 10        # bad fbits


def test_run_jobs_validation_on_host(mm):
    # mm_run_jobs validates the whole table on the host before anything launches
    L = mm.lib()
    assert L.mm_run_jobs(None, 0, None) == 0                       # nothing to do
    assert L.mm_run_jobs(None, 1, None) == 10                      # MM_E_ARG: null table
    bad = (mm._Job * 1)(mm._Job(7, 0, None, 0, 0, None, None, None, None, 0, 0))
    assert L.mm_run_jobs(bad, 1, None) == 10                       # unknown kind
    nullplan = (mm._Job * 1)(mm._Job(mm.Jobs.FORWARD, 0, None, 0, 0, None, None, None, None, 0, 0))
    assert L.mm_run_jobs(nullplan, 1, None) == 10                  # transform job without a plan
    big = (mm._Job * 1)(mm._Job(mm.Jobs.POLY_MUL, 0, None, 998244353, 3, 8, 8, 8, None, 4096, 4096))
    assert L.mm_run_jobs(big, 1, None) == 3                        # MM_E_UNSUPPORTED_SIZE: 8191 > 2^12
    nontt = (mm._Job * 1)(mm._Job(mm.Jobs.POLY_MUL, 0, None, 1000003, 2, 8, 8, 8, None, 100, 100))
    assert L.mm_run_jobs(nontt, 1, None) != 0                      # 2^8 does not divide p - 1
