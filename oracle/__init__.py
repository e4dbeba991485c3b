"""CPU oracle for arXiv 1407.3383's hot path -- TEST INFRASTRUCTURE ONLY.

Plain ctypes binding over ``oracle/oracle.c`` (u128 ``%`` arithmetic, the
definitions of P:889 / P:952 / P:973, schoolbook products).  Only ``tests/``,
``__graft_entry__.smoke()`` and ``bench.py``'s ``cpu_baseline`` / ``--impl
reference`` legs may import this package; the product package
``paper_1407_3383_b200`` never does, and this package imports nothing from it.

Parity status: every function exported here is pinned in
``tests/test_oracle.py`` against values fixed by the paper, SPEC.md worked
examples, closed forms, invariants or brute force.
"""
from __future__ import annotations

import ctypes
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "oracle.c")
_LIB = os.path.join(_HERE, "liboracle.so")

GOLDILOCKS = (1 << 64) - (1 << 32) + 1


def build(force: bool = False) -> str:
    """Compile oracle.c with gcc (host only)."""
    if force or not os.path.exists(_LIB) or os.path.getmtime(_LIB) < os.path.getmtime(_SRC):
        tmp = _LIB + f".tmp{os.getpid()}"
        subprocess.check_call(["gcc", "-O2", "-std=c11", "-shared", "-fPIC",
                               "-fvisibility=hidden", "-o", tmp, _SRC])
        os.replace(tmp, _LIB)
    return _LIB


_lib = None


def lib() -> ctypes.CDLL:
    global _lib
    if _lib is None:
        build()
        L = ctypes.CDLL(_LIB)
        u64, i32, sz = ctypes.c_uint64, ctypes.c_int, ctypes.c_size_t
        P = ctypes.c_void_p
        sig = {
            "or_addmod": (u64, [u64, u64, u64]),
            "or_submod": (u64, [u64, u64, u64]),
            "or_mulmod": (u64, [u64, u64, u64]),
            "or_powmod": (u64, [u64, u64, u64]),
            "or_is_prime": (i32, [u64]),
            "or_two_adicity": (i32, [u64]),
            "or_order_pow2": (u64, [u64, i32, u64]),
            "or_bitsize_r": (i32, [u64]),
            "or_barrett_params": (i32, [u64, i32, i32, P, P, P, P, P, P]),
            "or_reduce_barrett_fn6": (u64, [u64, u64, u64, i32, i32, u64, P]),
            "or_shoup_psi": (u64, [u64, u64, i32]),
            "or_montgomery_params": (i32, [u64, i32, P, P, P]),
            "or_reduce_montgomery_fn13": (u64, [u64, u64, u64, i32, u64]),
            "or_vec_addmod": (None, [P, P, P, sz, u64]),
            "or_vec_submod": (None, [P, P, P, sz, u64]),
            "or_vec_mulmod": (None, [P, P, P, sz, u64]),
            "or_vec_montmul": (None, [P, P, P, sz, u64, i32]),
            "or_vec_to_mont": (None, [P, P, sz, u64, i32]),
            "or_vec_shoup_psi": (None, [P, P, sz, u64, i32]),
            "or_bitrev": (u64, [u64, i32]),
            "or_root_of_unity": (u64, [u64, i32, u64]),
            "or_dft": (None, [P, P, sz, u64, u64]),
            "or_dft_point": (u64, [P, sz, u64, u64, u64]),
            "or_ntt": (None, [P, i32, u64, u64]),
            "or_intt": (None, [P, i32, u64, u64]),
            "or_to_bitrev": (None, [P, P, i32]),
            "or_algorithm1": (None, [P, P, i32, i32, u64, u64]),
            "or_poly_mul_schoolbook": (None, [P, sz, P, sz, P, u64]),
            "or_poly_mul_ntt": (i32, [P, sz, P, sz, P, u64, u64]),
            "or_poly_eval": (u64, [P, sz, u64, u64]),
            "or_carry_u16": (None, [P, sz, P, sz]),
            "or_int_mul_schoolbook_u16": (None, [P, sz, P, sz, P]),
            "or_int_mul_ntt_u16": (i32, [P, sz, P, sz, P, u64, u64]),
            "or_limbs_mod": (u64, [P, sz, u64]),
        }
        for name, (res, args) in sig.items():
            f = getattr(L, name)
            f.restype = res
            f.argtypes = args
        _lib = L
    return _lib


def _u64(a) -> np.ndarray:
    return np.ascontiguousarray(np.asarray(a, dtype=np.uint64))


def _u16(a) -> np.ndarray:
    return np.ascontiguousarray(np.asarray(a, dtype=np.uint16))


def _p(a: np.ndarray):
    return a.ctypes.data_as(ctypes.c_void_p)


# ---------------------------------------------------------------- scalars
def addmod(x, y, p):  return lib().or_addmod(x, y, p)
def submod(x, y, p):  return lib().or_submod(x, y, p)
def mulmod(x, y, p):  return lib().or_mulmod(x, y, p)
def powmod(b, e, p):  return lib().or_powmod(b, e, p)
def is_prime(n):      return bool(lib().or_is_prime(n))
def two_adicity(p):   return lib().or_two_adicity(p)
def order_pow2(w, k, p): return lib().or_order_pow2(w, k, p)
def bitsize_r(p):     return lib().or_bitsize_r(p)
def bitrev(i, k):     return lib().or_bitrev(i, k)
def root_of_unity(g, k, p): return lib().or_root_of_unity(g, k, p)
def shoup_psi(y, p, n=32): return lib().or_shoup_psi(y, p, n)


def barrett_params(p, n, profile):
    """Table 3. profile 2: m<=n-2, 1: m<=n-1, 0: m<=n."""
    outs = [ctypes.c_int() for _ in range(5)] + [ctypes.c_uint64()]
    rc = lib().or_barrett_params(p, n, profile, *[ctypes.byref(o) for o in outs])
    if rc != 0:
        raise ValueError(f"barrett_params rc={rc}")
    r, s, t, a, h, q = (o.value for o in outs)
    return dict(r=r, s=s, t=t, alpha_log2=a, h=h, q=q)


def reduce_barrett_fn6(a, p, s, t, q):
    it = ctypes.c_int()
    v = lib().or_reduce_barrett_fn6(a & (2**64 - 1), a >> 64, p, s, t, q, ctypes.byref(it))
    return v, it.value


def montgomery_params(p, m):
    chi, rho, r2 = ctypes.c_uint64(), ctypes.c_uint64(), ctypes.c_uint64()
    rc = lib().or_montgomery_params(p, m, ctypes.byref(chi), ctypes.byref(rho), ctypes.byref(r2))
    if rc != 0:
        raise ValueError(f"montgomery_params rc={rc}")
    return dict(chi=chi.value, rho=rho.value, r2=r2.value)


def reduce_montgomery_fn13(a, p, m, chi):
    return lib().or_reduce_montgomery_fn13(a & (2**64 - 1), a >> 64, p, m, chi)


# ---------------------------------------------------------------- vectors
def _vec2(name, x, y, p, *extra):
    x, y = _u64(x), _u64(y)
    z = np.empty_like(x)
    getattr(lib(), name)(_p(x), _p(y), _p(z), x.size, p, *extra)
    return z


def vec_addmod(x, y, p): return _vec2("or_vec_addmod", x, y, p)
def vec_submod(x, y, p): return _vec2("or_vec_submod", x, y, p)
def vec_mulmod(x, y, p): return _vec2("or_vec_mulmod", x, y, p)
def vec_montmul(x, y, p, m=32): return _vec2("or_vec_montmul", x, y, p, m)


def vec_to_mont(x, p, m=32):
    x = _u64(x); z = np.empty_like(x)
    lib().or_vec_to_mont(_p(x), _p(z), x.size, p, m)
    return z


def vec_shoup_psi(y, p, n=32):
    y = _u64(y); z = np.empty_like(y)
    lib().or_vec_shoup_psi(_p(y), _p(z), y.size, p, n)
    return z


# ---------------------------------------------------------------- NTT
def dft(a, w, p):
    a = _u64(a); out = np.empty_like(a)
    lib().or_dft(_p(a), _p(out), a.size, w, p)
    return out


def dft_point(a, w, i, p):
    a = _u64(a)
    return lib().or_dft_point(_p(a), a.size, w, i, p)


def _log2(n):
    k = int(n).bit_length() - 1
    if (1 << k) != n:
        raise ValueError("length must be a power of two")
    return k


def ntt(a, w, p):
    """Natural-order FFT_w by the textbook radix-2 algorithm."""
    a = _u64(a).copy()
    lib().or_ntt(_p(a), _log2(a.size), w, p)
    return a


def intt(a, w, p):
    a = _u64(a).copy()
    lib().or_intt(_p(a), _log2(a.size), w, p)
    return a


def to_bitrev(a):
    a = _u64(a); out = np.empty_like(a)
    lib().or_to_bitrev(_p(a), _p(out), _log2(a.size))
    return out


def ntt_rows(a, w, p, order="natural"):
    """Row-wise FFT_w of a 2-D array (rows are independent transforms)."""
    a = np.atleast_2d(_u64(a))
    out = np.empty_like(a)
    for r in range(a.shape[0]):
        v = ntt(a[r], w, p)
        out[r] = to_bitrev(v) if order == "bitrev" else v
    return out


def intt_rows(a, w, p, order="natural"):
    """Row-wise inverse; order = order of the INPUT spectrum."""
    a = np.atleast_2d(_u64(a))
    out = np.empty_like(a)
    for r in range(a.shape[0]):
        v = to_bitrev(a[r]) if order == "bitrev" else a[r]  # bitrev is an involution
        out[r] = intt(v, w, p)
    return out


def algorithm1(a, k1, w, p):
    a = _u64(a); out = np.empty_like(a)
    lib().or_algorithm1(_p(a), _p(out), _log2(a.size), k1, w, p)
    return out


# ---------------------------------------------------------------- products
def poly_mul_schoolbook(a, b, p):
    a, b = _u64(a), _u64(b)
    c = np.zeros(a.size + b.size - 1, dtype=np.uint64)
    lib().or_poly_mul_schoolbook(_p(a), a.size, _p(b), b.size, _p(c), p)
    return c


def poly_mul_ntt(a, b, p, g):
    a, b = _u64(a), _u64(b)
    c = np.zeros(a.size + b.size - 1, dtype=np.uint64)
    rc = lib().or_poly_mul_ntt(_p(a), a.size, _p(b), b.size, _p(c), p, g)
    if rc != 0:
        raise ValueError("transform length exceeds 2-adicity of p")
    return c


def poly_eval(a, x, p):
    a = _u64(a)
    return lib().or_poly_eval(_p(a), a.size, x, p)


def carry_u16(coef, nout):
    coef = _u64(coef)
    out = np.zeros(nout, dtype=np.uint16)
    lib().or_carry_u16(_p(coef), coef.size, _p(out), nout)
    return out


def int_mul_schoolbook_u16(a, b):
    a, b = _u16(a), _u16(b)
    c = np.zeros(a.size + b.size, dtype=np.uint16)
    lib().or_int_mul_schoolbook_u16(_p(a), a.size, _p(b), b.size, _p(c))
    return c


def int_mul_ntt_u16(a, b, p=GOLDILOCKS, g=7):
    a, b = _u16(a), _u16(b)
    c = np.zeros(a.size + b.size, dtype=np.uint16)
    rc = lib().or_int_mul_ntt_u16(_p(a), a.size, _p(b), b.size, _p(c), p, g)
    if rc != 0:
        raise ValueError("coefficient bound or 2-adicity exceeded")
    return c


def limbs_mod(a, q):
    a = _u16(a)
    return lib().or_limbs_mod(_p(a), a.size, q)


def poly_matmul_naive(A, B, p):
    """Polynomial matrix product by its definition: C[i][j] =
    sum_l A[i][l] B[l][j] in (Z/pZ)[x], every entry product a schoolbook
    product, sums mod p.  A: [m][kk][da], B: [kk][n][db] residues;
    returns [m][n][da + db - 1] (uint64)."""
    A, B = np.asarray(A), np.asarray(B)
    m, kk, da = A.shape
    kk2, n, db = B.shape
    if kk != kk2:
        raise ValueError("inner dimensions differ")
    C = np.zeros((m, n, da + db - 1), dtype=np.uint64)
    for i in range(m):
        for j in range(n):
            acc = np.zeros(da + db - 1, dtype=np.uint64)
            for l in range(kk):
                acc = vec_addmod(acc, poly_mul_schoolbook(A[i, l], B[l, j], p), p)
            C[i, j] = acc
    return C
