"""paper_1407_3383_b200 -- B200-native hot path of arXiv 1407.3383.

Thin Python binding over the C ABI in ``include/mmntt.h`` (``libmmntt.so``,
hand-written CUDA for sm_100a).  This module only marshals arguments: device
pointers of torch tensors, sizes, and the current CUDA stream.  Every step of
the path runs in the library's kernels; there is no CPU fallback -- if the
extension is missing or a call fails, an exception is raised.

Tensors: uint32 residues as ``torch.uint32`` (or int32 bit patterns), uint64
as ``torch.uint64`` (or int64), 16-bit limbs as ``torch.uint16`` (or int16).
"""
from __future__ import annotations

import ctypes
import os

import torch

from ._build import LIB as _LIB_PATH

__all__ = ["lib", "MMError", "Mod32", "Mod64", "ModF64", "ModNum", "Dist", "NttPlan", "poly_mul", "poly_mul_tft", "poly_matmul", "poly_mul_host", "int_mul_u16", "int_mul_u32", "int_matmul_u32", "Jobs", "GOLDILOCKS",
           "MUL_BARRETT", "MUL_SHOUP", "MUL_MONTGOMERY", "NATURAL", "BITREV", "EXPORTS"]

GOLDILOCKS = (1 << 64) - (1 << 32) + 1
MUL_BARRETT, MUL_SHOUP, MUL_MONTGOMERY = 0, 1, 2
NATURAL, BITREV = 0, 1
NUM_F14, NUM_F14_UP, NUM_F15_UP, NUM_F15_NEAR, NUM_F16, NUM_F16_UP = range(6)

_P = ctypes.c_void_p
_u32, _u64, _i32, _sz = ctypes.c_uint32, ctypes.c_uint64, ctypes.c_int, ctypes.c_size_t
_ST = ctypes.c_int

# every symbol declared in include/mmntt.h: name -> (restype, argtypes)
EXPORTS = {
    "mm_last_error": (ctypes.c_char_p, []),
    "mm_version": (ctypes.c_char_p, []),
    "mm_mod32_create": (_ST, [_u32, ctypes.POINTER(_P)]),
    "mm_mod32_destroy": (None, [_P]),
    "mm_modf64_create": (_ST, [_u64, ctypes.POINTER(_P)]),
    "mm_modf64_destroy": (None, [_P]),
    "mm_modadd_f64": (_ST, [_P, _P, _P, _P, _sz, _P]),
    "mm_modsub_f64": (_ST, [_P, _P, _P, _P, _sz, _P]),
    "mm_modmul_f64": (_ST, [_P, _P, _P, _P, _sz, _P]),
    "mm_mod32_info": (_ST, [_P, ctypes.POINTER(_u64)]),
    "mm_modadd_u32": (_ST, [_P, _P, _P, _P, _sz, _P]),
    "mm_modsub_u32": (_ST, [_P, _P, _P, _P, _sz, _P]),
    "mm_modmul_u32": (_ST, [_P, _i32, _P, _P, _P, _P, _sz, _P]),
    "mm_shoup_precompute_u32": (_ST, [_P, _P, _P, _sz, _P]),
    "mm_modop_u32_host": (_ST, [_P, _i32, _P, _P, _P, _P, _sz, _P]),
    "mm_to_mont_u32": (_ST, [_P, _P, _P, _sz, _P]),
    "mm_from_mont_u32": (_ST, [_P, _P, _P, _sz, _P]),
    "mm_ntt_plan_create": (_ST, [_i32, _u64, _i32, _u64, _sz, ctypes.POINTER(_P)]),
    "mm_ntt_plan_destroy": (None, [_P]),
    "mm_ntt_plan_info": (_ST, [_P, ctypes.POINTER(_u64)]),
    "mm_ntt_forward": (_ST, [_P, _P, _P, _i32, _P]),
    "mm_ntt_inverse": (_ST, [_P, _P, _P, _i32, _P]),
    "mm_ntt_forward_host": (_ST, [_P, _P, _P, _i32, _P]),
    "mm_ntt_inverse_host": (_ST, [_P, _P, _P, _i32, _P]),
    "mm_poly_mul": (_ST, [_i32, _u64, _u64, _P, _sz, _P, _sz, _P, _sz, _P]),
    "mm_poly_mul_tft": (_ST, [_u64, _u64, _P, _sz, _P, _sz, _P, _sz, _P]),
    "mm_poly_matmul": (_ST, [_u64, _u64, _P, _P, _P, _sz, _sz, _sz, _sz, _sz, _P]),
    "mm_int_matmul_u32": (_ST, [_P, _P, _P, _sz, _sz, _sz, _sz, _sz, _P]),
    "mm_int_mul_u32": (_ST, [_P, _sz, _P, _sz, _P, _P]),
    "mm_poly_mul_host": (_ST, [_i32, _u64, _u64, _P, _sz, _P, _sz, _P, _sz, _P]),
    "mm_poly_mul_ld": (_ST, [_i32, _u64, _u64, _P, _sz, _sz, _P, _sz, _sz, _P, _sz, _sz, _P]),
    "mm_int_mul_u16": (_ST, [_P, _sz, _P, _sz, _P, _P]),
    "mm_ntt_fwd_cols": (_ST, [_P, _P, _P, _sz, _sz, _P]),
    "mm_ntt_fwd_rows": (_ST, [_P, _P, _P, _sz, _sz, _P]),
    "mm_ntt_inv_rows": (_ST, [_P, _P, _P, _sz, _sz, _P]),
    "mm_ntt_inv_cols": (_ST, [_P, _P, _P, _sz, _sz, _P]),
    "mm_ipc_get_handle": (_ST, [_P, _P, ctypes.POINTER(_u64)]),
    "mm_ipc_open_handle": (_ST, [_P, ctypes.POINTER(_P)]),
    "mm_ipc_close": (_ST, [_P]),
    "mm_ntt_fwd_cols_p2p": (_ST, [_P, _P, _P, _i32, _i32, _sz, _sz, _P]),
    "mm_ntt_fwd_cols_u16": (_ST, [_P, _P, _sz, _P, _sz, _sz, _P]),
    "mm_ntt_pmul_rows_seg": (_ST, [_P, _P, _P, _P, _sz, _sz, _sz, _sz, _P]),
    "mm_carry_chunks_halo": (_ST, [_P, _sz, _sz, _P, _P]),
    "mm_carry_chunks_reduce": (_ST, [_P, _P, _sz, _sz, _sz, _sz, _sz, _sz, _i32, _P, _P]),
    "mm_carry_chunks_scan": (_ST, [_P, _sz, _sz, _P]),
    "mm_carry_chunks_apply": (_ST, [_P, _P, _sz, _sz, _sz, _sz, _sz, _sz, _i32, _P, _P, _P]),
    "mm_ntt_fwd_rows_seg": (_ST, [_P, _P, _P, _sz, _sz, _sz, _sz, _P]),
    "mm_ntt_inv_rows_seg": (_ST, [_P, _P, _P, _sz, _sz, _sz, _sz, _P]),
    "mm_launch_count": (ctypes.c_ulonglong, []),
    "mm_modnum_create": (_ST, [_i32, _u64, ctypes.POINTER(_P)]),
    "mm_modnum_destroy": (None, [_P]),
    "mm_modnum_info": (_ST, [_P, ctypes.POINTER(ctypes.c_double)]),
    "mm_mulmod_num": (_ST, [_P, _i32, _P, _P, _P, _sz, _P]),
    "mm_reduce_num": (_ST, [_P, _i32, _P, _P, _sz, _P]),
    "mm_mod64_create": (_ST, [_u64, ctypes.POINTER(_P)]),
    "mm_mod64_destroy": (None, [_P]),
    "mm_modadd_u64": (_ST, [_P, _P, _P, _P, _sz, _P]),
    "mm_modsub_u64": (_ST, [_P, _P, _P, _P, _sz, _P]),
    "mm_modmul_u64": (_ST, [_P, _P, _P, _P, _sz, _P]),
    "mm_dist_unique_id": (_ST, [_P]),
    "mm_dist_create": (_ST, [_P, _i32, _i32, ctypes.POINTER(_P)]),
    "mm_dist_destroy": (None, [_P]),
    "mm_dist_info": (_ST, [_P, ctypes.POINTER(ctypes.c_int64)]),
    "mm_dist_p2p_enable": (_ST, [_P, _sz]),
    "mm_dist_p2p_status": (_ST, [_P, ctypes.POINTER(_u64)]),
    "mm_ntt_forward_dist": (_ST, [_P, _P, _P, _P, _P]),
    "mm_ntt_inverse_dist": (_ST, [_P, _P, _P, _P, _P]),
    "mm_int_mul_u16_dist": (_ST, [_P, _P, _sz, _P, _sz, _P, _P]),
    "mm_int_mul_u16_dist_layout": (_ST, [_P, _sz, _sz, ctypes.POINTER(_u64)]),
    "mm_release_cached": (_ST, []),
    "mm_run_jobs": (_ST, [_P, _i32, _P]),
    "mm_set_product_streams": (_ST, [_i32]),
    "mm_probe_butterfly": (_ST, [_i32, _i32, ctypes.POINTER(ctypes.c_double), ctypes.POINTER(ctypes.c_double), _P]),
    "mm_probe_issue": (_ST, [_i32, _i32, ctypes.POINTER(ctypes.c_double), ctypes.POINTER(ctypes.c_double), _P]),
    "mm_prof_enable": (None, [_i32]),
    "mm_prof_collect": (_i32, [ctypes.c_char_p, _sz]),
}

STATUS = {0: "MM_OK", 1: "MM_E_INVALID_MODULUS", 2: "MM_E_PROFILE", 3: "MM_E_UNSUPPORTED_SIZE",
          4: "MM_E_BAD_ROOT", 5: "MM_E_RANGE", 6: "MM_E_SIZE_OVERFLOW", 7: "MM_E_ALIAS",
          8: "MM_E_CUDA", 9: "MM_E_NCCL", 10: "MM_E_ARG"}


class MMError(RuntimeError):
    def __init__(self, status: int, msg: str):
        super().__init__(f"{STATUS.get(status, status)}: {msg}")
        self.status = status


_lib = None


def lib() -> ctypes.CDLL:
    """Load libmmntt.so (built by __graft_entry__.build()). Raises if missing."""
    global _lib
    if _lib is None:
        if not os.path.exists(_LIB_PATH):
            raise ImportError(f"{_LIB_PATH} not built; run `python -c 'import __graft_entry__ as g; g.build()'`")
        L = ctypes.CDLL(_LIB_PATH)
        for name, (res, args) in EXPORTS.items():
            f = getattr(L, name)
            f.restype = res
            f.argtypes = args
        _lib = L
    return _lib


def _check(st: int):
    if st != 0:
        raise MMError(st, lib().mm_last_error().decode())


def _stream(t: torch.Tensor | None = None):
    dev = t.device if t is not None else torch.device("cuda")
    return ctypes.c_void_p(torch.cuda.current_stream(dev).cuda_stream)


def _ptr(t: torch.Tensor | None):
    if t is None:
        return None
    if not t.is_cuda:
        raise ValueError("tensors must live on a CUDA device (no CPU fallback)")
    if not t.is_contiguous():
        raise ValueError("tensors must be contiguous")
    return ctypes.c_void_p(t.data_ptr())


def _ptr_rows(t: torch.Tensor):
    """Pointer of a 2-D row-strided view (unit element stride; rows may be padded)."""
    if not t.is_cuda:
        raise ValueError("tensors must live on a CUDA device (no CPU fallback)")
    if t.dim() != 2 or t.stride(-1) != 1:
        raise ValueError("expected a 2-D view with unit element stride")
    return ctypes.c_void_p(t.data_ptr())


def _esz(t: torch.Tensor) -> int:
    return t.element_size()


def _need(t: torch.Tensor | None, numel: int, esize: int, name: str, like: torch.Tensor | None = None):
    """Argument check before a C call (the C ABI cannot see buffer lengths):
    a contiguous CUDA tensor of `numel` elements of `esize` bytes on the same
    device as `like`; raises ValueError otherwise."""
    if t is None:
        raise ValueError(f"{name} is required")
    if not t.is_cuda:
        raise ValueError(f"{name} must live on a CUDA device (no CPU fallback)")
    if like is not None and t.device != like.device:
        raise ValueError(f"{name} is on {t.device}, expected {like.device}")
    if t.element_size() != esize:
        raise ValueError(f"{name} must have {esize}-byte elements, got {t.element_size()}")
    if t.numel() != numel:
        raise ValueError(f"{name} must have {numel} elements, got {t.numel()}")
    if not t.is_contiguous():
        raise ValueError(f"{name} must be contiguous")
    return t


class _Job(ctypes.Structure):
    """mm_job (include/mmntt.h)."""
    _fields_ = [("kind", ctypes.c_int), ("order", ctypes.c_int), ("plan", _P), ("p", _u64), ("g", _u64),
                ("in_", _P), ("in2", _P), ("out", _P), ("out2", _P), ("la", _sz), ("lb", _sz)]


class Jobs:
    """Many small 32-bit problems in ONE launch (mm_run_jobs): transforms of
    one row of length n <= 2^12 (a single-pass NttPlan), forward-then-inverse
    round trips and polynomial products with la + lb - 1 <= 4096.  Add jobs,
    then ``run()`` on the current stream; the tensors and plans stay
    referenced until the builder is dropped or cleared."""
    FORWARD, INVERSE, ROUNDTRIP, POLY_MUL = range(4)

    def __init__(self):
        self._jobs: list[_Job] = []
        self._keep: list = []
        self._dev = None
        self._arr = None

    def _add(self, job: _Job, tensors, plan=None):
        if plan is not None:
            self._keep.append(plan)       # the C table holds the plan handle
        for t in tensors:
            if t is None:
                continue
            if self._dev is None:
                self._dev = t.device
            elif t.device != self._dev:
                raise ValueError(f"job tensor on {t.device}, expected {self._dev}")
        self._jobs.append(job)
        self._keep.extend(tensors)
        self._arr = None
        return self

    def _row(self, plan: "NttPlan", t, name):
        if plan.word_bits != 32:
            raise ValueError("jobs take 32-bit plans")
        return _need(t, plan.n, 4, name)

    def forward(self, plan: "NttPlan", x, out, order=BITREV):
        self._row(plan, x, "x"), self._row(plan, out, "out")
        return self._add(_Job(self.FORWARD, order, plan._h, 0, 0, _ptr(x), None, _ptr(out), None, 0, 0), (x, out), plan)

    def inverse(self, plan: "NttPlan", x, out, order=BITREV):
        self._row(plan, x, "x"), self._row(plan, out, "out")
        return self._add(_Job(self.INVERSE, order, plan._h, 0, 0, _ptr(x), None, _ptr(out), None, 0, 0), (x, out), plan)

    def roundtrip(self, plan: "NttPlan", x, out2, out=None, order=BITREV):
        """out = forward(x) in `order` (optional), out2 = inverse(forward(x))."""
        self._row(plan, x, "x"), self._row(plan, out2, "out2")
        if out is not None:
            self._row(plan, out, "out")
        return self._add(_Job(self.ROUNDTRIP, order, plan._h, 0, 0, _ptr(x), None, _ptr(out), _ptr(out2), 0, 0),
                         (x, out, out2), plan)

    def poly_mul(self, a, b, p: int, g: int, out):
        la, lb = a.numel(), b.numel()
        _need(a, la, 4, "a"), _need(b, lb, 4, "b", a), _need(out, la + lb - 1, 4, "out", a)
        return self._add(_Job(self.POLY_MUL, 0, None, int(p), int(g), _ptr(a), _ptr(b), _ptr(out), None, la, lb),
                         (a, b, out))

    def __len__(self):
        return len(self._jobs)

    def clear(self):
        self._jobs, self._keep, self._dev, self._arr = [], [], None, None

    def run(self):
        if not self._jobs:
            return
        if self._arr is None:
            self._arr = (_Job * len(self._jobs))(*self._jobs)
        s = ctypes.c_void_p(torch.cuda.current_stream(self._dev).cuda_stream)
        _check(lib().mm_run_jobs(self._arr, len(self._jobs), s))


# ------------------------------------------------------------------ modulus context
class ModF64:
    """Modulus context for residues held as IEEE doubles (mm_modf64_create,
    paper §3): odd p < 2^50, FMA-based products (Functions 16-18)."""

    def __init__(self, p: int):
        self.p = int(p)
        h = ctypes.c_void_p()
        _check(lib().mm_modf64_create(self.p, ctypes.byref(h)))
        self._h = h

    def __del__(self):
        h = getattr(self, "_h", None)
        if h and _lib is not None:
            _lib.mm_modf64_destroy(h)
            self._h = None

    def _run(self, name, x, y, out):
        if x.dtype != torch.float64 or y.dtype != torch.float64:
            raise ValueError("float64 residues expected")
        z = torch.empty_like(x) if out is None else out
        _need(y, x.numel(), 8, "y", x)
        _need(z, x.numel(), 8, "out", x)
        _check(getattr(lib(), name)(self._h, _ptr(x), _ptr(y), _ptr(z), x.numel(), _stream(x)))
        return z

    def add(self, x, y, out=None):
        return self._run("mm_modadd_f64", x, y, out)

    def sub(self, x, y, out=None):
        return self._run("mm_modsub_f64", x, y, out)

    def mul(self, x, y, out=None):
        return self._run("mm_modmul_f64", x, y, out)


class ModNum:
    """Numeric reductions (mm_modnum_create, paper §3.2-3.3, Functions 14-16):
    residues of an odd p held as integral float32 (fbits 32) or float64 (64)
    values; `variant` one of NUM_F14, NUM_F14_UP, NUM_F15_UP, NUM_F15_NEAR,
    NUM_F16, NUM_F16_UP (include/mmntt.h)."""

    def __init__(self, fbits: int, p: int):
        self.fbits, self.p = int(fbits), int(p)
        self.dtype = torch.float64 if fbits == 64 else torch.float32
        h = ctypes.c_void_p()
        _check(lib().mm_modnum_create(self.fbits, self.p, ctypes.byref(h)))
        self._h = h

    def __del__(self):
        h = getattr(self, "_h", None)
        if h and _lib is not None:
            _lib.mm_modnum_destroy(h)
            self._h = None

    def info(self) -> dict:
        out = (ctypes.c_double * 6)()
        _check(lib().mm_modnum_info(self._h, out))
        return dict(zip(["p", "u", "ubar", "l", "m", "fbits"], list(out)))

    def _chk(self, x, name):
        if x.dtype != self.dtype:
            raise ValueError(f"{name} must be {self.dtype}")

    def mul(self, x, y, variant=NUM_F16, out=None):
        self._chk(x, "x")
        self._chk(y, "y")
        z = torch.empty_like(x) if out is None else out
        _need(y, x.numel(), x.element_size(), "y", x)
        _need(z, x.numel(), x.element_size(), "out", x)
        _check(lib().mm_mulmod_num(self._h, int(variant), _ptr(x), _ptr(y), _ptr(z), x.numel(), _stream(x)))
        return z

    def reduce(self, a, variant=NUM_F14, out=None):
        self._chk(a, "a")
        z = torch.empty_like(a) if out is None else out
        _need(z, a.numel(), a.element_size(), "out", a)
        _check(lib().mm_reduce_num(self._h, int(variant), _ptr(a), _ptr(z), a.numel(), _stream(a)))
        return z


class Mod64:
    """64-bit modulus context (mm_mod64_create): p = 2^64 - 2^32 + 1 only."""

    def __init__(self, p: int = GOLDILOCKS):
        self.p = int(p)
        h = ctypes.c_void_p()
        _check(lib().mm_mod64_create(self.p, ctypes.byref(h)))
        self._h = h

    def __del__(self):
        h = getattr(self, "_h", None)
        if h and _lib is not None:
            _lib.mm_mod64_destroy(h)
            self._h = None

    def _run(self, name, x, y, out):
        if x.element_size() != 8:
            raise ValueError("64-bit residues expected")
        z = torch.empty_like(x) if out is None else out
        _need(y, x.numel(), 8, "y", x)
        _need(z, x.numel(), 8, "out", x)
        _check(getattr(lib(), name)(self._h, _ptr(x), _ptr(y), _ptr(z), x.numel(), _stream(x)))
        return z

    def add(self, x, y, out=None):
        return self._run("mm_modadd_u64", x, y, out)

    def sub(self, x, y, out=None):
        return self._run("mm_modsub_u64", x, y, out)

    def mul(self, x, y, out=None):
        return self._run("mm_modmul_u64", x, y, out)


class Mod32:
    """32-bit modulus context (mm_mod32_create): Table-3 Barrett profile and
    Montgomery constants precomputed once."""

    def __init__(self, p: int):
        self.p = int(p)
        h = ctypes.c_void_p()
        _check(lib().mm_mod32_create(self.p, ctypes.byref(h)))
        self._h = h

    def __del__(self):
        h = getattr(self, "_h", None)
        if h and _lib is not None:
            _lib.mm_mod32_destroy(h)
            self._h = None

    def info(self) -> dict:
        out = (ctypes.c_uint64 * 8)()
        _check(lib().mm_mod32_info(self._h, out))
        keys = ["p", "r", "s", "t", "h", "q", "pinv", "r2"]
        return dict(zip(keys, [int(v) for v in out]))

    def _out(self, x, out, *others):
        if x.element_size() != 4:
            raise ValueError("32-bit residues expected")
        z = torch.empty_like(x) if out is None else out
        _need(z, x.numel(), 4, "out", x)
        for nm, t in others:
            _need(t, x.numel(), 4, nm, x)
        return z

    def add(self, x, y, out=None):
        z = self._out(x, out, ("y", y))
        _check(lib().mm_modadd_u32(self._h, _ptr(x), _ptr(y), _ptr(z), x.numel(), _stream(x)))
        return z

    def sub(self, x, y, out=None):
        z = self._out(x, out, ("y", y))
        _check(lib().mm_modsub_u32(self._h, _ptr(x), _ptr(y), _ptr(z), x.numel(), _stream(x)))
        return z

    def mul(self, x, y, variant=MUL_MONTGOMERY, y_shoup=None, out=None):
        z = self._out(x, out, ("y", y), *((("y_shoup", y_shoup),) if variant == MUL_SHOUP else ()))
        _check(lib().mm_modmul_u32(self._h, variant, _ptr(x), _ptr(y), _ptr(y_shoup), _ptr(z), x.numel(),
                                   _stream(x)))
        return z

    def op_host(self, op: str, x, y, y_shoup=None, out=None):
        """add / sub / mul_barrett / mul_shoup / mul_montgomery on HOST uint32
        vectors (pinned for overlap) through mm_modop_u32_host's chunked upload /
        compute / download pipeline; returns after the result is in `out`."""
        code = {"add": 0, "sub": 1, "mul_barrett": 2, "mul_shoup": 3, "mul_montgomery": 4}[op]
        ts = [("x", x), ("y", y)] + ([("y_shoup", y_shoup)] if code == 3 else [])
        if out is None:
            out = torch.empty(x.shape, dtype=x.dtype, pin_memory=True)
        for nm, t in ts + [("out", out)]:
            if t is None or t.is_cuda or not t.is_contiguous() or t.numel() != x.numel() or t.element_size() != 4:
                raise ValueError(f"{nm} must be a contiguous host tensor of {x.numel()} 32-bit elements")
        st = torch.cuda.current_stream()
        vp = ctypes.c_void_p
        _check(lib().mm_modop_u32_host(self._h, code, vp(x.data_ptr()), vp(y.data_ptr()),
                                       vp(y_shoup.data_ptr()) if code == 3 else None, vp(out.data_ptr()), x.numel(),
                                       vp(st.cuda_stream)))
        st.synchronize()
        return out

    def shoup_precompute(self, y, out=None):
        z = self._out(y, out)
        _check(lib().mm_shoup_precompute_u32(self._h, _ptr(y), _ptr(z), y.numel(), _stream(y)))
        return z

    def to_mont(self, x, out=None):
        z = self._out(x, out)
        _check(lib().mm_to_mont_u32(self._h, _ptr(x), _ptr(z), x.numel(), _stream(x)))
        return z

    def from_mont(self, x, out=None):
        z = self._out(x, out)
        _check(lib().mm_from_mont_u32(self._h, _ptr(x), _ptr(z), x.numel(), _stream(x)))
        return z


# ------------------------------------------------------------------ NTT plans
class NttPlan:
    """Batched NTT of length 2^log2n over p with root omega (mm_ntt_plan_create).
    word_bits: 32 (uint32, p < 2^30), 64 (uint64, p = 2^64 - 2^32 + 1) or 52
    (float64 residues of an odd prime p < 2^50, FMA products, paper §3)."""

    def __init__(self, word_bits: int, p: int, log2n: int, omega: int, batch: int = 1):
        self.word_bits, self.p, self.log2n, self.omega, self.batch = word_bits, int(p), log2n, int(omega), batch
        self.n = 1 << log2n
        h = ctypes.c_void_p()
        _check(lib().mm_ntt_plan_create(word_bits, self.p, log2n, self.omega, batch, ctypes.byref(h)))
        self._h = h

    def __del__(self):
        h = getattr(self, "_h", None)
        if h and _lib is not None:
            _lib.mm_ntt_plan_destroy(h)
            self._h = None

    def info(self) -> dict:
        out = (ctypes.c_uint64 * 6)()
        _check(lib().mm_ntt_plan_info(self._h, out))
        return dict(n1=int(out[0]), n2=int(out[1]), passes=int(out[2]), ws_bytes=int(out[3]),
                    word_bits=int(out[4]), batch=int(out[5]))

    def _chk(self, x):
        if x.numel() != self.n * self.batch or _esz(x) * 8 != (32 if self.word_bits == 32 else 64):
            raise ValueError(f"expected {self.batch}x{self.n} elements of {self.word_bits} bits")

    def forward(self, x, out=None, order=BITREV):
        self._chk(x)
        out = x if out is None else out
        _need(out, x.numel(), x.element_size(), "out", x)
        _check(lib().mm_ntt_forward(self._h, _ptr(x), _ptr(out), order, _stream(x)))
        return out

    def inverse(self, x, out=None, order=BITREV):
        self._chk(x)
        out = x if out is None else out
        _need(out, x.numel(), x.element_size(), "out", x)
        _check(lib().mm_ntt_inverse(self._h, _ptr(x), _ptr(out), order, _stream(x)))
        return out

    def _host(self, fn, x, out, order):
        """HOST tensors (pinned for overlap) through the library's chunked upload /
        transform / download pipeline; returns after the result is in `out`."""
        if x.is_cuda:
            raise ValueError("forward_host / inverse_host take host tensors")
        self._chk(x)
        if not x.is_contiguous():
            raise ValueError("x must be contiguous")
        if out is None:
            out = torch.empty(x.shape, dtype=x.dtype, pin_memory=True)
        if out.is_cuda or not out.is_contiguous() or out.numel() != x.numel() or out.element_size() != x.element_size():
            raise ValueError("out must be a contiguous host tensor of x's size and element width")
        st = torch.cuda.current_stream()
        _check(fn(self._h, ctypes.c_void_p(x.data_ptr()), ctypes.c_void_p(out.data_ptr()), order,
                  ctypes.c_void_p(st.cuda_stream)))
        st.synchronize()
        return out

    def forward_host(self, x, out=None, order=BITREV):
        return self._host(lib().mm_ntt_forward_host, x, out, order)

    def inverse_host(self, x, out=None, order=BITREV):
        return self._host(lib().mm_ntt_inverse_host, x, out, order)

    # four-step building blocks (distributed transform)
    def fwd_cols(self, x, out, col0, ncols):
        _check(lib().mm_ntt_fwd_cols(self._h, _ptr(x), _ptr(out), col0, ncols, _stream(x)))
        return out

    def fwd_rows(self, x, out, row0, nrows):
        _check(lib().mm_ntt_fwd_rows(self._h, _ptr(x), _ptr(out), row0, nrows, _stream(x)))
        return out

    def inv_rows(self, x, out, row0, nrows):
        _check(lib().mm_ntt_inv_rows(self._h, _ptr(x), _ptr(out), row0, nrows, _stream(x)))
        return out

    def fwd_rows_seg(self, x, out, row0, nrows, seg_len, seg_stride):
        """Row pass reading segmented rows (an all-to-all receive buffer)."""
        _check(lib().mm_ntt_fwd_rows_seg(self._h, _ptr(x), _ptr(out), row0, nrows, seg_len, seg_stride, _stream(x)))
        return out

    def inv_rows_seg(self, x, out, row0, nrows, seg_len, seg_stride):
        """Inverse row pass writing segmented rows (an all-to-all send buffer)."""
        _check(lib().mm_ntt_inv_rows_seg(self._h, _ptr(x), _ptr(out), row0, nrows, seg_len, seg_stride, _stream(x)))
        return out

    def fwd_cols_p2p(self, x, peer_ptrs, rank, col0, ncols):
        """Column pass whose rows land directly in the peers' receive buffers
        (peer_ptrs: G device addresses; segment `rank` of each)."""
        arr = (ctypes.c_void_p * len(peer_ptrs))(*[int(q) for q in peer_ptrs])
        _check(lib().mm_ntt_fwd_cols_p2p(self._h, _ptr(x), arr, len(peer_ptrs), rank, col0, ncols, _stream(x)))

    def fwd_cols_u16(self, limbs, out, col0, ncols):
        """Steps 1-2 on columns [col0, col0 + ncols) of the zero-padded 16-bit limb
        vector viewed as [n2][n1] (widened to the 64-bit field); out [n2][ncols]."""
        _check(lib().mm_ntt_fwd_cols_u16(self._h, _ptr(limbs), limbs.numel(), _ptr(out), col0, ncols,
                                         _stream(limbs)))
        return out

    def pmul_rows_seg(self, a, b, out, row0, nrows, seg_len, seg_stride):
        """Rows of both operands (segmented receive buffers): steps 3-4, pointwise
        product, inverse steps 4-3 and twiddle, into a segmented send buffer
        (no n^-1: inv_cols applies it)."""
        _check(lib().mm_ntt_pmul_rows_seg(self._h, _ptr(a), _ptr(b), _ptr(out), row0, nrows, seg_len, seg_stride,
                                          _stream(a)))
        return out

    def inv_cols(self, x, out, col0, ncols):
        _check(lib().mm_ntt_inv_cols(self._h, _ptr(x), _ptr(out), col0, ncols, _stream(x)))
        return out


def set_product_streams(n: int):
    """Sub-batch concurrency of the batched products (mm_set_product_streams)."""
    _check(lib().mm_set_product_streams(int(n)))


def release_cached():
    """Free the library's cached plans and workspaces (mm_release_cached); synchronises."""
    _check(lib().mm_release_cached())


# ------------------------------------------------------------------ instrumentation
def launch_count() -> int:
    """Kernels launched by libmmntt so far in this process."""
    return int(lib().mm_launch_count())


def probe_butterfly(word_bits: int = 32, iters: int = 2000) -> float:
    """Register-only butterfly throughput of this GPU (butterflies / s)."""
    ms, bf = ctypes.c_double(), ctypes.c_double()
    _check(lib().mm_probe_butterfly(word_bits, iters, ctypes.byref(ms), ctypes.byref(bf), _stream()))
    return bf.value / (ms.value * 1e-3)


def probe_issue(kind: int, iters: int = 2000) -> float:
    """Warp instructions / s of one SASS class (0 IMAD, 1 IMAD.HI, 2 IADD3,
    3 VIADDMNMX, 4 IMAD.HI + 2 IADD3, 5 DFMA) over a full grid."""
    ms, ops = ctypes.c_double(), ctypes.c_double()
    _check(lib().mm_probe_issue(kind, iters, ctypes.byref(ms), ctypes.byref(ops), _stream()))
    return ops.value / (ms.value * 1e-3)


def prof_enable(on: bool = True):
    lib().mm_prof_enable(1 if on else 0)


def prof_collect() -> dict:
    """{kernel family: (launches, total_ms)} since the last collect (synchronises)."""
    n = lib().mm_prof_collect(None, 0)
    buf = ctypes.create_string_buffer(n + 1)
    lib().mm_prof_collect(buf, n + 1)
    out = {}
    for line in buf.value.decode().splitlines():
        name, cnt, ms = line.split()
        out[name] = (int(cnt), float(ms))
    return out


# ------------------------------------------------------------------ products
def _rows(t: torch.Tensor) -> torch.Tensor:
    """2-D view [rows, len] with unit element stride (row stride may exceed len)."""
    t2 = t if t.dim() == 2 else (t.reshape(1, -1) if t.dim() == 1 else t.reshape(-1, t.shape[-1]))
    if t2.stride(-1) != 1 or (t2.shape[0] > 1 and t2.stride(0) < t2.shape[1]):
        t2 = t2.contiguous()
    return t2


def poly_mul(a: torch.Tensor, b: torch.Tensor, p: int, g: int, word_bits: int | None = None,
             out: torch.Tensor | None = None) -> torch.Tensor:
    """Batched product mod p: a [batch, la], b [batch, lb] -> c [batch, la+lb-1].

    Row-strided 2-D views are passed through as leading dimensions
    (mm_poly_mul_ld), e.g. out = c_pad[:, :la+lb-1] of a [batch, ldc] tensor."""
    if word_bits is None:
        word_bits = 52 if a.dtype == torch.float64 else _esz(a) * 8
    a2, b2 = _rows(a), _rows(b)
    batch, la = a2.shape
    if b2.shape[0] != batch:
        raise ValueError("batch mismatch")
    lb = b2.shape[1]
    lc = la + lb - 1
    esz = 4 if word_bits == 32 else 8
    for nm, t in (("a", a), ("b", b)) + ((("out", out),) if out is not None else ()):
        if not t.is_cuda or t.device != a.device or t.element_size() != esz:
            raise ValueError(f"{nm} must be a CUDA tensor of {esz}-byte residues on {a.device}")
    if out is None:
        out = torch.empty((batch, lc), dtype=a.dtype, device=a.device)
    o2 = out if out.dim() == 2 else out.reshape(batch, lc)
    if tuple(o2.shape) != (batch, lc) or o2.stride(-1) != 1 or (batch > 1 and o2.stride(0) < lc):
        raise ValueError("out must be a [batch, la+lb-1] view with unit element stride")
    lda = a2.stride(0) if batch > 1 else la
    ldb = b2.stride(0) if batch > 1 else lb
    ldc = o2.stride(0) if batch > 1 else lc
    _check(lib().mm_poly_mul_ld(word_bits, int(p), int(g), _ptr_rows(a2), la, lda, _ptr_rows(b2), lb, ldb,
                                _ptr_rows(o2), ldc, batch, _stream(a)))
    return out if a.dim() > 1 else out.reshape(-1)


def poly_mul_tft(a: torch.Tensor, b: torch.Tensor, p: int, g: int, out: torch.Tensor | None = None) -> torch.Tensor:
    """Truncated-transform product mod p (mm_poly_mul_tft, Algorithm 1 with l < n):
    a [batch, la], b [batch, lb] uint32 -> c [batch, la + lb - 1]."""
    a2 = a.reshape(-1, a.shape[-1]) if a.dim() > 1 else a.reshape(1, -1)
    b2 = b.reshape(-1, b.shape[-1]) if b.dim() > 1 else b.reshape(1, -1)
    batch, la = a2.shape
    lb = b2.shape[1]
    if b2.shape[0] != batch or a.element_size() != 4:
        raise ValueError("a, b: [batch, la], [batch, lb] uint32")
    _need(b2, batch * lb, 4, "b", a)
    if out is None:
        out = torch.empty((batch, la + lb - 1), dtype=a.dtype, device=a.device)
    _need(out, batch * (la + lb - 1), 4, "out", a)
    _check(lib().mm_poly_mul_tft(int(p), int(g), _ptr(a2), la, _ptr(b2), lb, _ptr(out), batch, _stream(a)))
    return out if a.dim() > 1 else out.reshape(-1)


def poly_matmul(A: torch.Tensor, B: torch.Tensor, p: int, g: int, out: torch.Tensor | None = None) -> torch.Tensor:
    """Polynomial matrix product mod p (mm_poly_matmul):
    A [m, kk, da], B [kk, n, db] (uint32 residues) -> C [m, n, da + db - 1]."""
    if A.dim() != 3 or B.dim() != 3 or A.shape[1] != B.shape[0]:
        raise ValueError("expected A [m, kk, da] and B [kk, n, db]")
    m, kk, da = A.shape
    n, db = B.shape[1], B.shape[2]
    if A.element_size() != 4:
        raise ValueError("uint32 residues expected")
    _need(B, kk * n * db, 4, "B", A)
    if out is None:
        out = torch.empty((m, n, da + db - 1), dtype=A.dtype, device=A.device)
    _need(out, m * n * (da + db - 1), 4, "out", A)
    _check(lib().mm_poly_matmul(int(p), int(g), _ptr(A), _ptr(B), _ptr(out), m, kk, n, da, db, _stream(A)))
    return out


def poly_mul_host(a: torch.Tensor, b: torch.Tensor, p: int, g: int, out: torch.Tensor | None = None,
                  word_bits: int | None = None) -> torch.Tensor:
    """poly_mul on HOST tensors (pinned for overlap): mm_poly_mul_host pipelines
    chunked uploads, kernels and downloads; returns after the result is in
    `out` (synchronises the current stream)."""
    if a.is_cuda or b.is_cuda:
        raise ValueError("poly_mul_host takes host tensors")
    if word_bits is None:
        word_bits = 52 if a.dtype == torch.float64 else _esz(a) * 8
    a2 = a.reshape(-1, a.shape[-1]).contiguous()
    b2 = b.reshape(-1, b.shape[-1]).contiguous()
    batch, la = a2.shape
    lb = b2.shape[1]
    if out is None:
        out = torch.empty((batch, la + lb - 1), dtype=a.dtype, pin_memory=True)
    if out.is_cuda or not out.is_contiguous() or out.numel() != batch * (la + lb - 1):
        raise ValueError("out must be a contiguous host tensor of batch x (la + lb - 1)")
    st = torch.cuda.current_stream()
    _check(lib().mm_poly_mul_host(word_bits, int(p), int(g), ctypes.c_void_p(a2.data_ptr()), la,
                                  ctypes.c_void_p(b2.data_ptr()), lb, ctypes.c_void_p(out.data_ptr()), batch,
                                  ctypes.c_void_p(st.cuda_stream)))
    st.synchronize()
    return out


# ------------------------------------------------------------------ CUDA IPC (peer-scatter path)
def ipc_handle(t: torch.Tensor) -> tuple[bytes, int]:
    """(64-byte CUDA IPC handle of the allocation holding t, byte offset of t
    inside that allocation): the opener adds the offset to the opened base."""
    buf = ctypes.create_string_buffer(64)
    off = ctypes.c_uint64()
    _check(lib().mm_ipc_get_handle(ctypes.c_void_p(t.data_ptr()), buf, ctypes.byref(off)))
    return buf.raw, int(off.value)


def ipc_open(handle: bytes) -> int:
    """Open a peer allocation; returns its base address in this process."""
    ptr = ctypes.c_void_p()
    _check(lib().mm_ipc_open_handle(ctypes.create_string_buffer(handle, 64), ctypes.byref(ptr)))
    return int(ptr.value)


def ipc_close(ptr: int):
    _check(lib().mm_ipc_close(ctypes.c_void_p(ptr)))


# ------------------------------------------------------------------ chunked carries (sharded int_mul)
def carry_chunks_halo(coef, halo_out):
    """halo_out[r] = the last 4 coefficients of chunk r of a [nrows][c1] block."""
    _check(lib().mm_carry_chunks_halo(_ptr(coef), coef.shape[0], coef.shape[1], _ptr(halo_out), _stream(coef)))
    return halo_out


def carry_chunks_reduce(coef, halo, n1, col0, nc, nout, shift, agg):
    _check(lib().mm_carry_chunks_reduce(_ptr(coef), _ptr(halo), coef.shape[0], coef.shape[1], n1, col0, nc, nout,
                                        int(shift), _ptr(agg), _stream(coef)))
    return agg


def carry_chunks_scan(agg_all, G, nrows):
    _check(lib().mm_carry_chunks_scan(_ptr(agg_all), G, nrows, _stream(agg_all)))
    return agg_all


def carry_chunks_apply(coef, halo, n1, col0, nc, nout, shift, cin, out):
    _check(lib().mm_carry_chunks_apply(_ptr(coef), _ptr(halo), coef.shape[0], coef.shape[1], n1, col0, nc, nout,
                                       int(shift), _ptr(cin), _ptr(out), _stream(coef)))
    return out


def int_matmul_u32(A: torch.Tensor, B: torch.Tensor, out: torch.Tensor | None = None) -> torch.Tensor:
    """Integer matrix product (mm_int_matmul_u32): A [m, kk, na],
    B [kk, n, nb] 32-bit limbs -> C [m, n, na + nb + 1]."""
    if A.dim() != 3 or B.dim() != 3 or A.shape[1] != B.shape[0]:
        raise ValueError("expected A [m, kk, na] and B [kk, n, nb]")
    m, kk, na = A.shape
    n, nb = B.shape[1], B.shape[2]
    if A.element_size() != 4:
        raise ValueError("32-bit limbs expected")
    _need(B, kk * n * nb, 4, "B", A)
    if out is None:
        out = torch.empty((m, n, na + nb + 1), dtype=A.dtype, device=A.device)
    _need(out, m * n * (na + nb + 1), 4, "out", A)
    _check(lib().mm_int_matmul_u32(_ptr(A), _ptr(B), _ptr(out), m, kk, n, na, nb, _stream(A)))
    return out


def int_mul_u32(a: torch.Tensor, b: torch.Tensor, out: torch.Tensor | None = None) -> torch.Tensor:
    """Exact product of little-endian 32-bit limb arrays by the paper's three-prime
    FFT (mm_int_mul_u32); na + nb limbs."""
    if a.element_size() != 4 or b.element_size() != 4:
        raise ValueError("32-bit limbs expected")
    _need(b, b.numel(), 4, "b", a)
    if out is None:
        out = torch.empty(a.numel() + b.numel(), dtype=a.dtype, device=a.device)
    _need(out, a.numel() + b.numel(), 4, "out", a)
    _check(lib().mm_int_mul_u32(_ptr(a), a.numel(), _ptr(b), b.numel(), _ptr(out), _stream(a)))
    return out


def int_mul_u16(a: torch.Tensor, b: torch.Tensor, out: torch.Tensor | None = None) -> torch.Tensor:
    """Exact product of little-endian 16-bit limb arrays (mm_int_mul_u16); na + nb limbs."""
    if a.element_size() != 2:
        raise ValueError("16-bit limbs expected")
    _need(b, b.numel(), 2, "b", a)
    if out is None:
        out = torch.empty(a.numel() + b.numel(), dtype=a.dtype, device=a.device)
    _need(out, a.numel() + b.numel(), 2, "out", a)
    _check(lib().mm_int_mul_u16(_ptr(a), a.numel(), _ptr(b), b.numel(), _ptr(out), _stream(a)))
    return out


# ------------------------------------------------------------------ distributed (C ABI, NCCL inside the library)
class Dist:
    """Communicator of the library's distributed calls (mm_dist_create): rank 0
    draws an NCCL unique id (mm_dist_unique_id), torch.distributed broadcasts
    it, every rank builds the communicator on its current device."""

    def __init__(self, group=None):
        import torch.distributed as tdist
        self.rank = tdist.get_rank(group)
        self.world = tdist.get_world_size(group)
        idbuf = ctypes.create_string_buffer(128)
        if self.rank == 0:
            _check(lib().mm_dist_unique_id(idbuf))
        obj = [idbuf.raw if self.rank == 0 else None]
        src = tdist.get_global_rank(group, 0) if group is not None else 0
        tdist.broadcast_object_list(obj, src=src, group=group)
        h = ctypes.c_void_p()
        _check(lib().mm_dist_create(ctypes.create_string_buffer(obj[0], 128), self.rank, self.world, ctypes.byref(h)))
        self._h = h

    @classmethod
    def single(cls):
        """A one-rank communicator without a process group (tests, G = 1)."""
        self = cls.__new__(cls)
        self.rank, self.world = 0, 1
        idbuf = ctypes.create_string_buffer(128)
        _check(lib().mm_dist_unique_id(idbuf))
        h = ctypes.c_void_p()
        _check(lib().mm_dist_create(idbuf, 0, 1, ctypes.byref(h)))
        self._h = h
        return self

    def close(self):
        h = getattr(self, "_h", None)
        if h and _lib is not None:
            _lib.mm_dist_destroy(h)
            self._h = None

    def __del__(self):
        self.close()

    def info(self) -> dict:
        out = (ctypes.c_int64 * 4)()
        _check(lib().mm_dist_info(self._h, out))
        return dict(rank=int(out[0]), world=int(out[1]), p2p_bytes=int(out[2]), nccl_version=int(out[3]))

    def enable_p2p(self, nbytes: int):
        _check(lib().mm_dist_p2p_enable(self._h, int(nbytes)))

    def p2p_status(self) -> int:
        v = ctypes.c_uint64()
        _check(lib().mm_dist_p2p_status(self._h, ctypes.byref(v)))
        return int(v.value)

    def ntt_forward(self, plan: "NttPlan", x_cols: torch.Tensor, out: torch.Tensor | None = None) -> torch.Tensor:
        """Column block [n2, n1/G] (natural input) -> row block [n2/G, n1] of the TFT-order output."""
        inf = plan.info()
        n1, n2 = inf["n1"], inf["n2"]
        esz = 4 if plan.word_bits == 32 else 8
        _need(x_cols, n2 * (n1 // self.world), esz, "x_cols")
        if out is None:
            out = torch.empty((n2 // self.world, n1), dtype=x_cols.dtype, device=x_cols.device)
        _need(out, (n2 // self.world) * n1, esz, "out", x_cols)
        _check(lib().mm_ntt_forward_dist(self._h, plan._h, _ptr(x_cols), _ptr(out), _stream(x_cols)))
        return out

    def ntt_inverse(self, plan: "NttPlan", y_rows: torch.Tensor, out: torch.Tensor | None = None) -> torch.Tensor:
        inf = plan.info()
        n1, n2 = inf["n1"], inf["n2"]
        esz = 4 if plan.word_bits == 32 else 8
        _need(y_rows, (n2 // self.world) * n1, esz, "y_rows")
        if out is None:
            out = torch.empty((n2, n1 // self.world), dtype=y_rows.dtype, device=y_rows.device)
        _need(out, n2 * (n1 // self.world), esz, "out", y_rows)
        _check(lib().mm_ntt_inverse_dist(self._h, plan._h, _ptr(y_rows), _ptr(out), _stream(y_rows)))
        return out

    def int_mul_layout(self, na: int, nb: int) -> dict:
        out = (ctypes.c_uint64 * 4)()
        _check(lib().mm_int_mul_u16_dist_layout(self._h, na, nb, out))
        return dict(n1=int(out[0]), n2=int(out[1]), c1=int(out[2]), log2n=int(out[3]))

    def int_mul_u16(self, a: torch.Tensor, b: torch.Tensor, out: torch.Tensor | None = None) -> torch.Tensor:
        """Sharded a b (16-bit limbs, whole on every rank) -> this rank's [n2, c1]
        limb block (limb r n1 + rank c1 + i at (r, i))."""
        if a.element_size() != 2:
            raise ValueError("16-bit limbs expected")
        _need(b, b.numel(), 2, "b", a)
        L = self.int_mul_layout(a.numel(), b.numel())
        if out is None:
            out = torch.empty((L["n2"], L["c1"]), dtype=a.dtype, device=a.device)
        _need(out, L["n2"] * L["c1"], 2, "out", a)
        _check(lib().mm_int_mul_u16_dist(self._h, _ptr(a), a.numel(), _ptr(b), b.numel(), _ptr(out), _stream(a)))
        return out
