"""GPU parity: the CUDA path (through the C ABI) vs the CPU oracle, bit-exact.

Inputs come from gen/ (seeded, shared by both sides).  Sizes span several
tiles and a ragged tail; the BASELINE full-size configs are checked on
sampled outputs (or properties that hold at any size) in the launch
configuration bench.py uses.
"""
import os
import random

import numpy as np
import pytest

torch = pytest.importorskip("torch")

import gen
from gen import config_seed, limbs16, residues

pytestmark = pytest.mark.gpu

P30 = 998244353
P32 = 3221225473
PG = (1 << 64) - (1 << 32) + 1
DEV = "cuda"


@pytest.fixture(scope="module")
def mm():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import paper_1407_3383_b200 as m
    m.lib()
    return m


def dev(a):
    return torch.from_numpy(np.ascontiguousarray(a)).to(DEV)


def host(t):
    return t.cpu().numpy()


def u64(a):
    return np.asarray(a).astype(np.uint64)


# ------------------------------------------------------------------ C2 elementwise
def test_mod32_info(mm, O):
    for p in (P32, P30, 65537, 2147483647, 7):
        info = mm.Mod32(p).info()
        prof = 2 if info["r"] <= 30 else (1 if info["r"] <= 31 else 0)
        bp = O.barrett_params(p, 32, prof)
        assert (info["s"], info["t"], info["h"], info["q"]) == (bp["s"], bp["t"], bp["h"], bp["q"])
        mp = O.montgomery_params(p, 32)
        assert (info["pinv"] * p) % (1 << 32) == 1
        assert (mp["chi"] * p + 1) % (1 << 32) == 0          # chi = -p^-1 mod 2^32
        assert info["r2"] == pow(2, 64, p)


def _ew_check(mm, O, p, x, y, offset=0):
    M = mm.Mod32(p)
    xt, yt = dev(x), dev(y)
    if offset:
        xt, yt = xt[offset:], yt[offset:]
        x, y = x[offset:], y[offset:]
    xs, ys = u64(x), u64(y)
    assert np.array_equal(u64(host(M.add(xt, yt))), O.vec_addmod(xs, ys, p))
    assert np.array_equal(u64(host(M.sub(xt, yt))), O.vec_submod(xs, ys, p))
    ref = O.vec_mulmod(xs, ys, p)
    assert np.array_equal(u64(host(M.mul(xt, yt, mm.MUL_BARRETT))), ref)
    ysh = M.shoup_precompute(yt)
    assert np.array_equal(u64(host(ysh)), O.vec_shoup_psi(ys, p, 32))
    assert np.array_equal(u64(host(M.mul(xt, yt, mm.MUL_SHOUP, y_shoup=ysh))), ref)
    assert np.array_equal(u64(host(M.mul(xt, yt, mm.MUL_MONTGOMERY))), O.vec_montmul(xs, ys, p, 32))
    xm = M.to_mont(xt)
    assert np.array_equal(u64(host(xm)), O.vec_to_mont(xs, p, 32))
    assert np.array_equal(host(M.from_mont(xm)), host(xt))


@pytest.mark.parametrize("p", [P32, P30, 2147483647, 65537])
def test_elementwise_random(mm, O, p):
    n = (1 << 20) + 3                         # many CTAs + ragged tail
    x = residues(config_seed(2), 1, n, p)
    y = residues(config_seed(2), 2, n, p)
    _ew_check(mm, O, p, x, y)
    _ew_check(mm, O, p, x, y, offset=1)        # unaligned pointers: scalar path


@pytest.mark.parametrize("p", [P32, P30, 7])
def test_elementwise_boundary(mm, O, p):
    B = sorted({0, 1, 2, (p - 1) // 2, (p + 1) // 2, p - 2, p - 1, min(p - 1, 1 << 31), min(p - 1, (1 << 32) // 3)})
    x = np.array([a for a in B for _ in B], dtype=np.uint32)
    y = np.array([b for _ in B for b in B], dtype=np.uint32)
    _ew_check(mm, O, p, x, y)


def test_elementwise_inplace_and_empty(mm, O):
    M = mm.Mod32(P32)
    x = residues(3, 1, 1000, P32)
    y = residues(3, 2, 1000, P32)
    xt, yt = dev(x), dev(y)
    M.add(xt, yt, out=xt)
    assert np.array_equal(u64(host(xt)), O.vec_addmod(u64(x), u64(y), P32))
    e = torch.empty(0, dtype=torch.uint32, device=DEV)
    M.mul(e, e)


@pytest.mark.slow
def test_elementwise_full_c2_all(mm, O):
    # BASELINE C2 at full size: every one of the 2^28 outputs of every operation
    # against the oracle (2^24-element chunks checked on host threads)
    from concurrent.futures import ThreadPoolExecutor
    p, n, CH = P32, 1 << 28, 1 << 24
    x = gen.residues_torch(config_seed(2), 1, n, p, DEV).view(torch.uint32)
    y = gen.residues_torch(config_seed(2), 2, n, p, DEV).view(torch.uint32)
    M = mm.Mod32(p)
    ysh = M.shoup_precompute(y)
    xh = u64(host(x.view(torch.int32)).view(np.uint32))
    yh = u64(host(y.view(torch.int32)).view(np.uint32))
    ops = [("add", lambda: M.add(x, y), lambda a, b: O.vec_addmod(a, b, p)),
           ("sub", lambda: M.sub(x, y), lambda a, b: O.vec_submod(a, b, p)),
           ("mont", lambda: M.mul(x, y, mm.MUL_MONTGOMERY), lambda a, b: O.vec_montmul(a, b, p, 32)),
           ("barrett", lambda: M.mul(x, y, mm.MUL_BARRETT), lambda a, b: O.vec_mulmod(a, b, p)),
           ("shoup", lambda: M.mul(x, y, mm.MUL_SHOUP, y_shoup=ysh), lambda a, b: O.vec_mulmod(a, b, p)),
           ("shoup_psi", lambda: ysh, lambda a, b: O.vec_shoup_psi(b, p, 32))]
    nt = max(1, min(32, os.cpu_count() or 1))
    for name, gpu, ref in ops:
        z = u64(host(gpu().view(torch.int32)).view(np.uint32))

        def ok(i):
            sl = slice(i * CH, (i + 1) * CH)
            return np.array_equal(z[sl], ref(xh[sl], yh[sl]))
        with ThreadPoolExecutor(nt) as ex:
            res = list(ex.map(ok, range(n // CH)))
        assert all(res), (name, [i for i, r in enumerate(res) if not r][:5])
        del z


def test_elementwise_full_c2_sampled(mm, O):
    # BASELINE C2: 2^28 uint32 pairs, p = 3221225473, bench launch config
    p, n = P32, 1 << 28
    x = gen.residues_torch(config_seed(2), 1, n, p, DEV).view(torch.uint32)
    y = gen.residues_torch(config_seed(2), 2, n, p, DEV).view(torch.uint32)
    M = mm.Mod32(p)
    idx = np.sort(np.random.default_rng(0).choice(n, 1 << 16, replace=False))
    it = torch.from_numpy(idx).to(DEV)

    def pick(t):      # gather sampled outputs (int32 view: indexing is not defined for uint32 on CUDA)
        return u64(host(t.view(torch.int32)[it]).view(np.uint32))

    xs = pick(x)
    ys = pick(y)
    assert np.array_equal(xs, u64(residues(config_seed(2), 1, n, p)[idx]))   # generator parity host/device
    for name, z, ref in [("add", M.add(x, y), O.vec_addmod(xs, ys, p)),
                         ("sub", M.sub(x, y), O.vec_submod(xs, ys, p)),
                         ("mont", M.mul(x, y, mm.MUL_MONTGOMERY), O.vec_montmul(xs, ys, p, 32)),
                         ("barrett", M.mul(x, y, mm.MUL_BARRETT), O.vec_mulmod(xs, ys, p))]:
        assert np.array_equal(pick(z), ref), name
        del z
    ysh = M.shoup_precompute(y)
    assert np.array_equal(pick(ysh), O.vec_shoup_psi(ys, p, 32))
    z = M.mul(x, y, mm.MUL_SHOUP, y_shoup=ysh)
    assert np.array_equal(pick(z), O.vec_mulmod(xs, ys, p))


# ------------------------------------------------------------------ FP64 reduction (paper §3)
P50 = 1108307720798209          # 63 2^44 + 1, Table 12's prime


@pytest.mark.parametrize("p", [P50, (1 << 50) - 27, P30, 7])
def test_modf64(mm, O, p):
    # Functions 16-18 over doubles vs the oracle (u128 %), random + boundary residues
    n = (1 << 18) + 3
    x = residues(config_seed(2), 7, n, p)
    y = residues(config_seed(2), 8, n, p)
    B = sorted({0, 1, 2, (p - 1) // 2, (p + 1) // 2, p - 2, p - 1})
    x = np.concatenate([x, np.array([a for a in B for _ in B], dtype=np.uint64)])
    y = np.concatenate([y, np.array([b for _ in B for b in B], dtype=np.uint64)])
    M = mm.ModF64(p)
    xt = torch.from_numpy(x.astype(np.float64)).to(DEV)
    yt = torch.from_numpy(y.astype(np.float64)).to(DEV)
    for op, ref in [(M.add, O.vec_addmod(x, y, p)), (M.sub, O.vec_submod(x, y, p)), (M.mul, O.vec_mulmod(x, y, p))]:
        z = host(op(xt, yt))
        assert np.array_equal(z, np.floor(z)), "non-integral result"
        assert np.array_equal(z.astype(np.uint64), ref)
    z = host(M.mul(xt[1:], yt[1:]))           # unaligned vectors: scalar tail path
    assert np.array_equal(z.astype(np.uint64), O.vec_mulmod(x[1:], y[1:], p))


def test_modf64_rejects_wide_prime(mm):
    with pytest.raises(Exception):
        mm.ModF64((1 << 61) - 1)


def test_mod64_goldilocks(mm, O):
    # mm_mod64_create + vector add / sub / mul over p = 2^64 - 2^32 + 1 vs u128 %
    n = (1 << 19) + 3
    x = residues(config_seed(4), 11, n, PG)
    y = residues(config_seed(4), 12, n, PG)
    B = sorted({0, 1, 2, (1 << 32) - 1, 1 << 32, (1 << 32) + 1, 1 << 63, (PG - 1) // 2, PG - (1 << 32), PG - 2, PG - 1})
    x = np.concatenate([x, np.array([a for a in B for _ in B], dtype=np.uint64)])
    y = np.concatenate([y, np.array([b for _ in B for b in B], dtype=np.uint64)])
    M = mm.Mod64()
    xt, yt = dev(x), dev(y)
    for op, ref in [(M.add, O.vec_addmod(x, y, PG)), (M.sub, O.vec_submod(x, y, PG)), (M.mul, O.vec_mulmod(x, y, PG))]:
        assert np.array_equal(host(op(xt, yt)), ref)
        assert np.array_equal(host(op(xt[1:], yt[1:])), ref[1:])      # unaligned: scalar tail kernel
    with pytest.raises(mm.MMError):
        mm.Mod64(P30)


# ------------------------------------------------------------------ numeric reductions (paper §3.2-3.3)
# (fbits, p, variants): primes at the bit bounds of Table 10 (float m = 11, 21;
# double m = 25, 26, 50) and small ones; each variant only where its bound allows
_NUM_CASES = [
    (64, 67108859, (0, 1, 4, 5)),            # m = 26 = l/2: Function 14 (+ u-bar), Function 16
    (64, 33554393, (0, 1, 2, 3, 4, 5)),      # m = 25 = (l-1)/2: Functions 14, 15, 16
    (64, 65537, (0, 1, 2, 3, 4, 5)),
    (64, 1125899906842597, (4, 5)),          # m = 50 = l - 2: Function 16 only
    (64, P50, (4, 5)),
    (32, 2039, (0, 1, 2, 3, 4, 5)),          # float, m = 11
    (32, 2097143, (4, 5)),                   # float, m = 21 = l - 2
    (32, 7, (0, 1, 2, 3, 4, 5)),
]


@pytest.mark.parametrize("fbits,p,variants", _NUM_CASES)
def test_numeric_mulmod(mm, O, fbits, p, variants):
    # Functions 14 / 15 / 16 and their toward-+inf forms vs the oracle's (x y) rem p
    from fractions import Fraction
    M = mm.ModNum(fbits, p)
    inf = M.info()
    assert Fraction(inf["ubar"]) >= Fraction(1, p) and Fraction(inf["u"]) == Fraction(1.0 / p if fbits == 64 else float(np.float32(1) / np.float32(p)))
    dt = np.float64 if fbits == 64 else np.float32
    n = (1 << 18) + 5
    x = residues(config_seed(2), 20 + fbits, n, p)
    y = residues(config_seed(2), 21 + fbits, n, p)
    B = sorted({0, 1, 2, (p - 1) // 2, (p + 1) // 2, p - 2, p - 1})
    x = np.concatenate([x, np.array([a for a in B for _ in B], dtype=np.uint64)])
    y = np.concatenate([y, np.array([b for _ in B for b in B], dtype=np.uint64)])
    ref = O.vec_mulmod(x, y, p)
    xt, yt = dev(x.astype(dt)), dev(y.astype(dt))
    for v in variants:
        z = host(M.mul(xt, yt, variant=v))
        assert np.array_equal(z, np.floor(z)), (p, v)
        assert np.array_equal(z.astype(np.uint64), ref), (fbits, p, v)
        z = host(M.mul(xt[1:], yt[1:], variant=v))            # unaligned: scalar tail kernel
        assert np.array_equal(z.astype(np.uint64), ref[1:]), (fbits, p, v, "unaligned")
    for v in set(range(6)) - set(variants):                    # beyond the variant's bound m
        with pytest.raises(mm.MMError):
            M.mul(xt, yt, variant=v)


@pytest.mark.parametrize("fbits,p,variants", [c for c in _NUM_CASES if set(c[2]) & {0, 1, 2}])
def test_numeric_reduce(mm, O, fbits, p, variants):
    # Functions 14 / 15 on integers a < alpha p (alpha = 2^(l/2), 2^floor((l-1)/2))
    M = mm.ModNum(fbits, p)
    l = 52 if fbits == 64 else 23
    dt = np.float64 if fbits == 64 else np.float32
    rng = np.random.default_rng(fbits + p % 1000)
    for v in [v for v in variants if v in (0, 1, 2)]:
        alpha = 1 << (l // 2 if v in (0, 1) else (l - 1) // 2)
        top = alpha * p
        a = rng.integers(0, top, (1 << 16) + 3, dtype=np.uint64)
        edge = [0, 1, p - 1, p, p + 1, 2 * p - 1, 2 * p, top - 1, top - p, top - p - 1, (alpha - 1) * p, alpha * p // 2]
        a = np.concatenate([a, np.array(edge, dtype=np.uint64)])
        z = host(M.reduce(dev(a.astype(dt)), variant=v))
        assert np.array_equal(z.astype(np.uint64), O.vec_mulmod(a, np.ones_like(a), p)), (fbits, p, v)
    at = dev(np.zeros(8, dtype=dt))
    for v in (3, 4, 5):                                        # F15_NEAR needs products; F16 two factors
        with pytest.raises(mm.MMError):
            M.reduce(at, variant=v)


# ------------------------------------------------------------------ NTT
def _ntt_roundtrip(mm, O, bits, p, g, k, batch, seed=5):
    w = O.root_of_unity(g, k, p)
    x = residues(seed, k, batch << k, p).reshape(batch, 1 << k)
    plan = mm.NttPlan(bits, p, k, w, batch)
    xt = dev(x)
    nat = O.ntt_rows(x, w, p)
    bit = np.stack([O.to_bitrev(r) for r in nat])
    yb = plan.forward(xt, out=torch.empty_like(xt), order=mm.BITREV)
    assert np.array_equal(u64(host(yb)), bit), (bits, k, "bitrev")
    yn = plan.forward(xt, out=torch.empty_like(xt), order=mm.NATURAL)
    assert np.array_equal(u64(host(yn)), nat), (bits, k, "natural")
    assert np.array_equal(host(plan.inverse(yb.clone(), order=mm.BITREV)), x)
    assert np.array_equal(host(plan.inverse(yn.clone(), order=mm.NATURAL)), x)
    # in place
    xt2 = xt.clone()
    plan.forward(xt2, order=mm.BITREV)
    assert np.array_equal(u64(host(xt2)), bit)


@pytest.mark.parametrize("k", list(range(1, 17)) + [18, 20])
def test_ntt32_sizes(mm, O, k):
    _ntt_roundtrip(mm, O, 32, P30, 3, k, batch=3 if k < 18 else 1)


@pytest.mark.parametrize("k", list(range(1, 17)) + [18, 20])
def test_ntt64_sizes(mm, O, k):
    _ntt_roundtrip(mm, O, 64, PG, 7, k, batch=3 if k < 18 else 1)


def _f64_roundtrip(mm, O, p, g, k, batch):
    w = O.root_of_unity(g, k, p)
    x = residues(9, k, batch << k, p).reshape(batch, 1 << k)
    plan = mm.NttPlan(52, p, k, w, batch)
    xt = torch.from_numpy(x.astype(np.float64)).to(DEV)
    nat = O.ntt_rows(x, w, p)
    yn = host(plan.forward(xt, out=torch.empty_like(xt), order=mm.NATURAL))
    assert np.array_equal(yn.astype(np.uint64), nat), (k, "natural")
    yb = plan.forward(xt, out=torch.empty_like(xt), order=mm.BITREV)
    assert np.array_equal(host(yb).astype(np.uint64), np.stack([O.to_bitrev(r) for r in nat])), (k, "bitrev")
    assert np.array_equal(host(plan.inverse(yb.clone(), order=mm.BITREV)).astype(np.uint64), x)


@pytest.mark.parametrize("k", [1, 2, 5, 10, 12, 13, 16, 18, 20])
def test_ntt_f64_sizes(mm, O, k):
    # Table 12's prime 63 2^44 + 1 (generator 11) with FP64 residues (paper §3)
    _f64_roundtrip(mm, O, P50, 11, k, batch=3 if k < 18 else 1)


def test_poly_mul_f64(mm, O):
    for la, lb, batch in [(1, 1, 1), (511, 513, 2), (3000, 5000, 1), (1 << 15, 1 << 15, 1)]:
        a = residues(la, 1, la * batch, P50).reshape(batch, la)
        b = residues(lb, 2, lb * batch, P50).reshape(batch, lb)
        c = host(mm.poly_mul(torch.from_numpy(a.astype(np.float64)).to(DEV),
                             torch.from_numpy(b.astype(np.float64)).to(DEV), P50, 11))
        for r in range(batch):
            ref = O.poly_mul_schoolbook(a[r], b[r], P50) if la * lb <= 1 << 22 else O.poly_mul_ntt(a[r], b[r], P50, 11)
            assert np.array_equal(c[r].astype(np.uint64), ref), (la, lb, r)


@pytest.mark.parametrize("bits,p,g", [(32, P30, 3), (32, 469762049, 3), (64, PG, 7)])
def test_ntt_edge_rows(mm, O, bits, p, g):
    for k in (4, 10, 14):
        n = 1 << k
        w = O.root_of_unity(g, k, p)
        x = np.zeros((4, n), dtype=np.uint32 if bits == 32 else np.uint64)
        x[0, 0] = 1                 # delta -> all ones (BASELINE)
        x[1, :] = p - 1             # constant p-1 -> (n (p-1), 0, ...)
        x[3, 1] = 1                 # delta_1 -> w^i
        plan = mm.NttPlan(bits, p, k, w, 4)
        y = u64(host(plan.forward(dev(x), order=mm.NATURAL)))
        assert (y[0] == 1).all()
        assert y[1, 0] == (n * (p - 1)) % p and not y[1, 1:].any()
        assert not y[2].any()
        assert [int(v) for v in y[3, :8]] == [pow(w, i, p) for i in range(8)]


def test_ntt_c1_batch(mm, O):
    # BASELINE C1: 16 independent fwd+inv NTTs of length 2^10 over 998244353
    p, k = P30, 10
    w = O.root_of_unity(3, k, p)
    assert O.order_pow2(w, k, p) == 1 << k
    x = residues(config_seed(1), 1, 16 << k, p).reshape(16, 1 << k)
    plan = mm.NttPlan(32, p, k, w, 16)
    y = plan.forward(dev(x), order=mm.NATURAL)
    assert np.array_equal(u64(host(y)), O.ntt_rows(x, w, p))
    assert np.array_equal(host(plan.inverse(y, order=mm.NATURAL)), x)


def test_ntt_c3_forward_full(mm, O):
    # BASELINE C3 forward: 4096 x 2^16 over 998244353, every row against the
    # oracle's textbook NTT (host threads over rows), TFT and natural order
    from concurrent.futures import ThreadPoolExecutor
    p, k, B = P30, 16, 4096
    w = O.root_of_unity(3, k, p)
    x = gen.residues_torch(config_seed(3), 1, B << k, p, DEV).view(torch.uint32).reshape(B, 1 << k)
    plan = mm.NttPlan(32, p, k, w, B)
    yb = host(plan.forward(x, out=torch.empty_like(x), order=mm.BITREV))
    yn = host(plan.forward(x, out=torch.empty_like(x), order=mm.NATURAL))
    xh = host(x)

    def bad_rows(rows):
        out = []
        for r in rows:
            nat = O.ntt(u64(xh[r]), w, p)
            if not (np.array_equal(u64(yn[r]), nat) and np.array_equal(u64(yb[r]), O.to_bitrev(nat))):
                out.append(r)
        return out
    nt = max(1, min(32, os.cpu_count() or 1))
    with ThreadPoolExecutor(nt) as ex:
        bad = sum(ex.map(bad_rows, [range(t, B, nt) for t in range(nt)]), [])
    assert not bad, bad[:10]


def test_ntt_c4_sampled(mm, O):
    # BASELINE C4: 8 transforms of 2^24 over Goldilocks, four-step (2^13 x 2^11 here)
    k, B = 24, 8
    w = O.root_of_unity(7, k, PG)
    x = gen.residues_torch(config_seed(4), 1, B << k, PG, DEV).view(torch.uint64).reshape(B, 1 << k)
    plan = mm.NttPlan(64, PG, k, w, B)
    inf = plan.info()
    assert inf["n1"] * inf["n2"] == 1 << k and inf["passes"] == 2
    y = plan.forward(x, out=torch.empty_like(x), order=mm.BITREV)
    rng = np.random.default_rng(4)
    for b in (0, 7):
        xb = host(x[b])
        for pos in [0, 1, (1 << k) - 1] + list(rng.integers(0, 1 << k, 2)):
            i = O.bitrev(int(pos), k)
            assert int(host(y[b, int(pos)])) == O.dft_point(xb, w, i, PG), (b, pos)
    z = plan.inverse(y, order=mm.BITREV)
    assert torch.equal(z.view(torch.int64), x.view(torch.int64))


@pytest.mark.slow
def test_ntt_c4_full(mm, O):
    # BASELINE C4 at full size: all 8 transforms of 2^24 compared element by
    # element with the oracle's textbook NTT in both output orders, in the
    # bench launch configuration (batch 8: the 2^13-row x 2^11-column four-step
    # with the full 2^24 step-2 table, sub-batches on the fork streams); the
    # oracle transforms run on host threads (~10 s each)
    from concurrent.futures import ThreadPoolExecutor
    k, B = 24, 8
    w = O.root_of_unity(7, k, PG)
    x = gen.residues_torch(config_seed(4), 1, B << k, PG, DEV).view(torch.uint64).reshape(B, 1 << k)
    plan = mm.NttPlan(64, PG, k, w, B)
    xh = host(x)
    with ThreadPoolExecutor(B) as ex:
        nat = list(ex.map(lambda t: O.ntt(xh[t], w, PG), range(B)))
    yb = plan.forward(x, out=torch.empty_like(x), order=mm.BITREV)
    ybh = host(yb)
    for t in range(B):
        assert np.array_equal(ybh[t], O.to_bitrev(nat[t])), t
    del yb
    yn = plan.forward(x, out=torch.empty_like(x), order=mm.NATURAL)
    ynh = host(yn)
    for t in range(B):
        assert np.array_equal(ynh[t], nat[t]), t
    z = plan.inverse(yn, out=torch.empty_like(yn), order=mm.NATURAL)
    assert torch.equal(z.view(torch.int64), x.view(torch.int64))


@pytest.mark.slow
def test_ntt64_2e25_full(mm, O):
    # 2^25 Goldilocks transforms from 64-bit words: 2^13 columns of 2^12 points
    # whose step-2 twiddles w^(j1 k) are formed on chip from per-column bases
    # (T_lo[k mod 64] T_hi[k / 64], ColsK::OTF; C5 reaches the same tiles from
    # 16-bit limbs), batch 2 so the sub-batches run on the fork streams; every
    # output against the oracle's textbook NTT, then the round trip
    from concurrent.futures import ThreadPoolExecutor
    k, B = 25, 2
    w = O.root_of_unity(7, k, PG)
    x = gen.residues_torch(config_seed(4), 3, B << k, PG, DEV).view(torch.uint64).reshape(B, 1 << k)
    plan = mm.NttPlan(64, PG, k, w, B)
    inf = plan.info()
    assert inf["n2"] == 1 << 12 and inf["n1"] == 1 << 13, inf
    xh = host(x)
    with ThreadPoolExecutor(B) as ex:
        nat = list(ex.map(lambda t: O.ntt(xh[t], w, PG), range(B)))
    yb = plan.forward(x, out=torch.empty_like(x), order=mm.BITREV)
    ybh = host(yb)
    for t in range(B):
        assert np.array_equal(ybh[t], O.to_bitrev(nat[t])), t
    z = plan.inverse(yb, out=torch.empty_like(yb), order=mm.BITREV)
    assert torch.equal(z.view(torch.int64), x.view(torch.int64))


@pytest.mark.parametrize("k", [10, 11, 12, 20, 22, 23])
@pytest.mark.parametrize("e", [1, 3, 65])
def test_ntt64_gold_and_generic_tiles(mm, O, k, e):
    # 2^11 / 2^12 / 2^13 Goldilocks tiles run gold.cuh when w^(n/64) = 2^39 (e = 1,
    # and e = 65 = 1 mod 64 gives the same 64-th root), the generic radix-8 groups
    # otherwise (e = 3); every path must equal the definition (oracle NTT)
    w = pow(O.root_of_unity(7, k, PG), e, PG)
    batch = 3 if k < 16 else 1
    x = residues(6, k, batch << k, PG).reshape(batch, 1 << k)
    plan = mm.NttPlan(64, PG, k, w, batch)
    xt = dev(x)
    nat = O.ntt_rows(x, w, PG)
    yb = plan.forward(xt, out=torch.empty_like(xt), order=mm.BITREV)
    assert np.array_equal(u64(host(yb)), np.stack([O.to_bitrev(r) for r in nat])), (k, e)
    assert np.array_equal(host(plan.inverse(yb.clone(), order=mm.BITREV)), x), (k, e)


@pytest.mark.parametrize("k", [10, 11, 12, 13, 20, 24])
def test_ntt64_gold_extreme_rows(mm, O, k):
    # closed forms through the Goldilocks tiles: delta_0 -> ones, constant p - 1 ->
    # (n (p-1), 0, ...), zeros -> zeros, delta_1 -> w^i; the all-(p-1) row drives
    # every 3-word intermediate of gold.cuh to its largest values
    n = 1 << k
    w = O.root_of_unity(7, k, PG)
    x = torch.zeros((4, n), dtype=torch.int64, device=DEV)
    x[0, 0] = 1
    x[1, :] = PG - 1 - (1 << 64)    # p - 1 as the int64 bit pattern
    x[3, 1] = 1
    plan = mm.NttPlan(64, PG, k, w, 4)
    y = plan.forward(x, out=torch.empty_like(x), order=mm.NATURAL)
    assert bool((y[0] == 1).all())
    assert int(y[1, 0]) & ((1 << 64) - 1) == (n * (PG - 1)) % PG and not bool(y[1, 1:].any())
    assert not bool(y[2].any())
    assert [int(v) & ((1 << 64) - 1) for v in host(y[3, :8])] == [pow(w, i, PG) for i in range(8)]
    z = plan.inverse(y, order=mm.NATURAL)
    assert torch.equal(z, x)


# ------------------------------------------------------------------ poly_mul
def test_poly_mul_c1(mm, O):
    p, g = P30, 3
    a = residues(config_seed(1), 1, 512, p)
    b = residues(config_seed(1), 2, 512, p)
    c = mm.poly_mul(dev(a), dev(b), p, g)
    assert np.array_equal(u64(host(c)), O.poly_mul_schoolbook(a, b, p))


@pytest.mark.parametrize("bits,p,g", [(32, P30, 3), (32, 469762049, 3), (64, PG, 7)])
def test_poly_mul_ragged(mm, O, bits, p, g):
    rng = random.Random(bits)
    cases = [(1, 1, 1), (1, 7, 2), (3, 2, 5), (511, 513, 3), (1000, 24, 2), (2049, 2048, 2), (3000, 5000, 2),
             (1 << 13, 1 << 13, 1), (12345, 777, 1)]
    for la, lb, batch in cases:
        a = residues(rng.randrange(1 << 30), 1, la * batch, p).reshape(batch, la)
        b = residues(rng.randrange(1 << 30), 2, lb * batch, p).reshape(batch, lb)
        c = u64(host(mm.poly_mul(dev(a), dev(b), p, g, word_bits=bits)))
        for r in range(batch):
            ref = O.poly_mul_schoolbook(a[r], b[r], p) if la * lb <= 1 << 22 else O.poly_mul_ntt(a[r], b[r], p, g)
            assert np.array_equal(c[r], ref), (la, lb, r)


@pytest.mark.parametrize("p,g", [(P30, 3), (469762049, 3)])
def test_poly_mul_fast16_shapes(mm, O, p, g):
    # every product length in (2^15, 2^16] runs the specialised 256 x 256
    # passes: half-zero / full / ragged inputs, exact and truncated outputs
    cases = [(1 << 15, 1 << 15, 3), (30001, 20000, 2), (40000, 20000, 2), (1 << 16, 1, 1), (1, 1 << 16, 1),
             (32769, 32768, 1), (16385, 16384, 2)]
    rng = random.Random(p)
    for la, lb, batch in cases:
        a = residues(rng.randrange(1 << 30), 1, la * batch, p).reshape(batch, la)
        b = residues(rng.randrange(1 << 30), 2, lb * batch, p).reshape(batch, lb)
        c = u64(host(mm.poly_mul(dev(a), dev(b), p, g)))
        for r in range(batch):
            assert np.array_equal(c[r], O.poly_mul_ntt(a[r], b[r], p, g)), (la, lb, r)
    # leading dimensions: strided a / b rows and a padded output (mm_poly_mul_ld)
    for la, lb, lda, ldb, ldc in [(1 << 15, 1 << 15, (1 << 15) + 4, 1 << 16, 1 << 16), (3000, 5000, 3001, 5003, 8000),
                                  (30001, 20000, 30008, 20000, 50016)]:
        batch = 3
        A = residues(la + 7, 1, batch * lda, p).reshape(batch, lda)
        B = residues(lb + 7, 2, batch * ldb, p).reshape(batch, ldb)
        Cp = torch.full((batch, ldc), 0xDEADBEEF, dtype=torch.uint32, device=DEV)
        mm.poly_mul(dev(A)[:, :la], dev(B)[:, :lb], p, g, out=Cp[:, :la + lb - 1])
        ch = host(Cp)
        for r in range(batch):
            assert np.array_equal(u64(ch[r, :la + lb - 1]), O.poly_mul_ntt(A[r, :la], B[r, :lb], p, g)), (la, lb, r)
            assert (ch[r, la + lb - 1:] == 0xDEADBEEF).all(), "wrote beyond the row"
    # extreme residues: all p-1 (every lazy range at its maximum)
    a = np.full((2, 1 << 15), p - 1, dtype=np.uint32)
    c = u64(host(mm.poly_mul(dev(a), dev(a), p, g)))
    for r in range(2):
        assert np.array_equal(c[r], O.poly_mul_ntt(a[r], a[r], p, g))


def test_poly_mul_host_pipeline(mm, O):
    # host operands, several pipeline chunks (~192 products each) + a ragged last chunk
    p, g, B, d = P30, 3, 500, 1 << 15
    a = torch.from_numpy(residues(11, 1, B * d, p).reshape(B, d)).pin_memory()
    b = torch.from_numpy(residues(11, 2, B * d, p).reshape(B, d)).pin_memory()
    c = mm.poly_mul_host(a, b, p, g)
    cd = mm.poly_mul(a.to(DEV), b.to(DEV), p, g).cpu()
    assert torch.equal(c, cd)
    for r in (0, 191, 192, 499):
        assert np.array_equal(u64(c[r].numpy()), O.poly_mul_ntt(a[r].numpy(), b[r].numpy(), p, g)), r
    # small and 64-bit: a single chunk
    a = residues(12, 1, 3 * 700, PG).reshape(3, 700)
    b = residues(12, 2, 3 * 300, PG).reshape(3, 300)
    c = mm.poly_mul_host(torch.from_numpy(a), torch.from_numpy(b), PG, 7)
    for r in range(3):
        assert np.array_equal(u64(c[r].numpy()), O.poly_mul_schoolbook(a[r], b[r], PG)), r


def test_poly_mul_host_back_to_back(mm, O):
    # consecutive calls of 2, 1, 4 and 3 chunks: the slot rotation continues
    # across calls (a call's first upload takes the slot after the previous
    # call's last one); every result checked
    p, g, d = P30, 3, 1 << 15
    outs = []
    for i, B in enumerate((300, 100, 700, 450)):
        a = torch.from_numpy(residues(40 + i, 1, B * d, p).reshape(B, d)).pin_memory()
        b = torch.from_numpy(residues(40 + i, 2, B * d, p).reshape(B, d)).pin_memory()
        c = torch.empty((B, 2 * d - 1), dtype=torch.uint32).pin_memory()
        mm.poly_mul_host(a, b, p, g, out=c)
        outs.append((a, b, c))
    torch.cuda.synchronize()
    for a, b, c in outs:
        assert torch.equal(c, mm.poly_mul(a.to(DEV), b.to(DEV), p, g).cpu())
    a, b, c = outs[2]
    for r in (0, 191, 192, 699):
        assert np.array_equal(u64(c[r].numpy()), O.poly_mul_ntt(a[r].numpy(), b[r].numpy(), p, g)), r


def test_onepass_2e13_32bit(mm, O):
    # 32-bit transforms and products of 2^13 points run in one pass (a 32 KiB
    # row tile): a batch spanning several tiles with a ragged tail, both orders,
    # round trips, and ragged products whose length lands in (2^12, 2^13]
    p, g, k, B = P30, 3, 13, 37
    w = O.root_of_unity(g, k, p)
    plan = mm.NttPlan(32, p, k, w, B)
    assert plan.info()["passes"] == 1
    x = residues(81, 1, B << k, p).reshape(B, 1 << k)
    xt = dev(x)
    nat = O.ntt_rows(x, w, p)
    yb = plan.forward(xt, out=torch.empty_like(xt), order=mm.BITREV)
    assert np.array_equal(u64(host(yb)), np.stack([O.to_bitrev(r) for r in nat]))
    yn = plan.forward(xt, out=torch.empty_like(xt), order=mm.NATURAL)
    assert np.array_equal(u64(host(yn)), nat)
    assert np.array_equal(host(plan.inverse(yb, order=mm.BITREV)), x)
    assert np.array_equal(host(plan.inverse(yn, order=mm.NATURAL)), x)
    for la, lb, batch in ((4096, 4097, 5), (8000, 193, 3), (2049, 2049, 19), (1, 8192, 2), (4096, 1, 2)):
        a = residues(82 + la, 1, batch * la, p).reshape(batch, la)
        b = residues(82 + la, 2, batch * lb, p).reshape(batch, lb)
        c = u64(host(mm.poly_mul(dev(a), dev(b), p, g)))
        for r in range(batch):
            assert np.array_equal(c[r], O.poly_mul_ntt(a[r], b[r], p, g)), (la, lb, r)
    # all p - 1: every lazy range at its maximum
    a = np.full((2, 4096), p - 1, dtype=np.uint32)
    c = u64(host(mm.poly_mul(dev(a), dev(a), p, g)))
    assert np.array_equal(c[0], O.poly_mul_ntt(a[0], a[0], p, g)) and np.array_equal(c[1], c[0])


def test_modop_host_pipeline(mm, O):
    # mm_modop_u32_host: 2^24 + 5 elements (three chunks of 2^23 for the
    # three-array operations, a ragged tail), every operation against the device
    # call and sampled against the oracle; in place on the host; empty vectors
    p, n = 3221225473, (1 << 24) + 5
    x = torch.from_numpy(residues(71, 1, n, p)).pin_memory()
    y = torch.from_numpy(residues(71, 2, n, p)).pin_memory()
    M = mm.Mod32(p)
    xd, yd = x.to(DEV), y.to(DEV)
    ys = M.shoup_precompute(yd).cpu().pin_memory()
    idx = np.concatenate([np.arange(0, 64), np.arange((1 << 23) - 32, (1 << 23) + 32), np.arange(n - 64, n)])
    xs, ysm = u64(x.numpy()[idx]), u64(y.numpy()[idx])
    want = {"add": (M.add(xd, yd), O.vec_addmod(xs, ysm, p)), "sub": (M.sub(xd, yd), O.vec_submod(xs, ysm, p)),
            "mul_barrett": (M.mul(xd, yd, mm.MUL_BARRETT), O.vec_mulmod(xs, ysm, p)),
            "mul_shoup": (M.mul(xd, yd, mm.MUL_SHOUP, y_shoup=ys.to(DEV)), O.vec_mulmod(xs, ysm, p)),
            "mul_montgomery": (M.mul(xd, yd, mm.MUL_MONTGOMERY), O.vec_montmul(xs, ysm, p, 32))}
    for op, (zd, zo) in want.items():
        z = M.op_host(op, x, y, y_shoup=ys)
        assert torch.equal(z, zd.cpu()), op
        assert np.array_equal(u64(z.numpy()[idx]), zo), op
    z = x.clone().pin_memory()
    M.op_host("mul_barrett", z, y, out=z)
    assert torch.equal(z, want["mul_barrett"][0].cpu())
    e = torch.empty(0, dtype=torch.uint32)
    assert M.op_host("add", e, e).numel() == 0
    with pytest.raises(ValueError):
        M.op_host("mul_shoup", x, y)
    with pytest.raises(ValueError):
        M.op_host("add", xd, y)


def test_ntt_host_pipeline(mm, O):
    # mm_ntt_forward_host / mm_ntt_inverse_host: host rows through the three-slot
    # upload / transform / download pipeline.  500 rows of 2^16 (192 rows per
    # chunk: two full chunks and a ragged one), both orders, in place on the host
    p, k, B = P30, 16, 500
    w = O.root_of_unity(3, k, p)
    x = torch.from_numpy(residues(61, 1, B << k, p).reshape(B, 1 << k)).pin_memory()
    plan = mm.NttPlan(32, p, k, w, B)
    for order in (mm.BITREV, mm.NATURAL):
        y = plan.forward_host(x, order=order)
        assert torch.equal(y, plan.forward(x.to(DEV), out=torch.empty_like(x, device=DEV), order=order).cpu())
        for r in (0, 191, 192, 383, 384, 499):
            nat = O.ntt(u64(x[r].numpy()), w, p)
            assert np.array_equal(u64(y[r].numpy()), nat if order == mm.NATURAL else O.to_bitrev(nat)), (order, r)
        z = y.clone().pin_memory()
        plan.inverse_host(z, out=z, order=order)
        assert torch.equal(z, x), order
    # Goldilocks, 9 rows of 2^20 (6 rows per chunk), every row against the oracle
    k, B = 20, 9
    w = O.root_of_unity(7, k, PG)
    xh = residues(62, 1, B << k, PG).reshape(B, 1 << k)
    plan64 = mm.NttPlan(64, PG, k, w, B)
    y = plan64.forward_host(torch.from_numpy(xh).pin_memory(), order=mm.BITREV).numpy()
    for r in range(B):
        assert np.array_equal(u64(y[r]), O.to_bitrev(O.ntt(xh[r], w, PG))), r
    # a single transform is one chunk
    plan1 = mm.NttPlan(64, PG, k, w, 1)
    y1 = plan1.forward_host(torch.from_numpy(xh[4:5].copy()), order=mm.BITREV).numpy()
    assert np.array_equal(y1[0], y[4])
    with pytest.raises(ValueError):
        plan1.forward_host(dev(xh[:1]))


def test_host_pipeline_mixed_calls(mm, O):
    # a host product and a host transform queued back to back through the C ABI
    # without a synchronise in between: the two calls cut the library's slots
    # differently (the second call's uploads must wait for every pending
    # download of the first)
    import ctypes
    p, g, d, B = P30, 3, 1 << 15, 450
    a = torch.from_numpy(residues(63, 1, B * d, p).reshape(B, d)).pin_memory()
    b = torch.from_numpy(residues(63, 2, B * d, p).reshape(B, d)).pin_memory()
    c = torch.empty((B, 2 * d - 1), dtype=torch.uint32).pin_memory()
    k, Bn = 12, 5000
    w = O.root_of_unity(3, k, p)
    x = torch.from_numpy(residues(64, 1, Bn << k, p).reshape(Bn, 1 << k)).pin_memory()
    y = torch.empty_like(x).pin_memory()
    plan = mm.NttPlan(32, p, k, w, Bn)
    c.fill_(0)
    y.fill_(0)
    torch.cuda.synchronize()
    L, vp = mm.lib(), ctypes.c_void_p
    st = torch.cuda.current_stream()
    for _ in range(2):
        assert L.mm_poly_mul_host(32, p, g, vp(a.data_ptr()), d, vp(b.data_ptr()), d, vp(c.data_ptr()), B,
                                  vp(st.cuda_stream)) == 0
        assert L.mm_ntt_forward_host(plan._h, vp(x.data_ptr()), vp(y.data_ptr()), mm.BITREV, vp(st.cuda_stream)) == 0
    st.synchronize()
    assert torch.equal(c, mm.poly_mul(a.to(DEV), b.to(DEV), p, g).cpu())
    assert torch.equal(y, plan.forward(x.to(DEV), out=torch.empty_like(x, device=DEV), order=mm.BITREV).cpu())
    for r in (0, 4999):
        assert np.array_equal(u64(y[r].numpy()), O.to_bitrev(O.ntt(u64(x[r].numpy()), w, p))), r


@pytest.mark.parametrize("p,g", [(P30, 3), (469762049, 3)])
def test_poly_mul_tft(mm, O, p, g):
    # Algorithm 1 with l < n (truncated rows) + inverse column TFT: products of
    # every length class -- lambda = 1, small, just over a power of two, full
    rng = random.Random(p + 1)
    cases = [(2049, 2049, 2), (4097, 1, 1), (2500, 2000, 3), (1 << 15, 3, 2), ((1 << 15) + 1, 1 << 15, 1),
             (40000, 30000, 1), (30001, 20000, 2), (1 << 16, 1 << 16, 1), (70000, 60001, 1), (3, 5000, 2)]
    for la, lb, batch in cases:
        a = residues(rng.randrange(1 << 30), 1, la * batch, p).reshape(batch, la)
        b = residues(rng.randrange(1 << 30), 2, lb * batch, p).reshape(batch, lb)
        c = u64(host(mm.poly_mul_tft(dev(a), dev(b), p, g)))
        cp = u64(host(mm.poly_mul(dev(a), dev(b), p, g)))
        assert np.array_equal(c, cp), (la, lb)
        for r in range(min(batch, 2)):
            ref = O.poly_mul_schoolbook(a[r], b[r], p) if la * lb <= 1 << 22 else O.poly_mul_ntt(a[r], b[r], p, g)
            assert np.array_equal(c[r], ref), (la, lb, r)
    # maximal residues
    a = np.full((1, 33000), p - 1, dtype=np.uint32)
    c = u64(host(mm.poly_mul_tft(dev(a), dev(a), p, g)))
    assert np.array_equal(c[0], O.poly_mul_ntt(a[0], a[0], p, g))


def test_poly_mul_c3_small_batch(mm, O):
    p, g = P30, 3
    B, d = 8, 1 << 15
    a = residues(config_seed(3), 1, B * d, p).reshape(B, d)
    b = residues(config_seed(3), 2, B * d, p).reshape(B, d)
    c = u64(host(mm.poly_mul(dev(a), dev(b), p, g)))
    for r in range(B):
        assert np.array_equal(c[r], O.poly_mul_ntt(a[r], b[r], p, g)), r


def test_poly_mul_c3_full(mm, O):
    # BASELINE C3 product: 4096 pairs of degree < 2^15 (bench launch config);
    # every row checked by c(r) = a(r) b(r) at a random point and in full.
    p, g, B, d = P30, 3, 4096, 1 << 15
    a = gen.residues_torch(config_seed(3), 1, B * d, p, DEV).view(torch.uint32).reshape(B, d)
    b = gen.residues_torch(config_seed(3), 2, B * d, p, DEV).view(torch.uint32).reshape(B, d)
    # bench.py's launch: output rows at leading dimension 2^16 (mm_poly_mul_ld)
    c_pad = torch.empty((B, 1 << 16), dtype=torch.uint32, device=DEV)
    c = mm.poly_mul(a, b, p, g, out=c_pad[:, :2 * d - 1])
    ah, bh, ch = host(a), host(b), host(c)
    cp = mm.poly_mul(a[:64], b[:64], p, g)                # packed layout, same products
    assert torch.equal(c[:64], cp)
    rng = random.Random(3)
    for r in range(0, B, 1):
        x = rng.randrange(1, p)
        assert O.poly_eval(ch[r], x, p) == O.mulmod(O.poly_eval(ah[r], x, p), O.poly_eval(bh[r], x, p), p), r
    # every one of the 4096 products element by element against the oracle's NTT
    # product (threads over rows: the ctypes calls release the GIL)
    from concurrent.futures import ThreadPoolExecutor

    def bad_rows(rows):
        return [r for r in rows if not np.array_equal(u64(ch[r]), O.poly_mul_ntt(ah[r], bh[r], p, g))]
    nt = max(1, min(32, os.cpu_count() or 1))
    with ThreadPoolExecutor(nt) as ex:
        bad = sum(ex.map(bad_rows, [range(t, B, nt) for t in range(nt)]), [])
    assert not bad, bad[:10]


# ------------------------------------------------------------------ polynomial matrix product
@pytest.mark.parametrize("m,kk,n,da,db,p,g", [(3, 3, 3, 8, 8, 469762049, 3), (1, 1, 1, 1, 1, P30, 3),
                                              (4, 5, 3, 100, 37, P30, 3), (2, 3, 2, 3000, 2000, 469762049, 3),
                                              (5, 2, 7, 33, 1, P30, 3)])
def test_poly_matmul(mm, O, m, kk, n, da, db, p, g):
    # P:962-969 vs the naive matrix of schoolbook products (single-pass and four-step sizes)
    A = residues(m * 100 + da, 1, m * kk * da, p).reshape(m, kk, da)
    B = residues(n * 100 + db, 2, kk * n * db, p).reshape(kk, n, db)
    C = u64(host(mm.poly_matmul(dev(A), dev(B), p, g)))
    assert np.array_equal(C, O.poly_matmul_naive(A, B, p))


def test_poly_matmul_table15_sampled(mm, O):
    # Table 15 shape: 32 x 32 matrices, degrees < 2^15 over 469762049; every entry
    # checked by evaluation at a random point (C(r) = A(r) B(r) as matrices over Z/pZ)
    p, g, N, d = 469762049, 3, 32, 1 << 15
    A = gen.residues_torch(15, 1, N * N * d, p, DEV).view(torch.uint32).reshape(N, N, d)
    B = gen.residues_torch(15, 2, N * N * d, p, DEV).view(torch.uint32).reshape(N, N, d)
    C = host(mm.poly_matmul(A, B, p, g))
    Ah, Bh = host(A), host(B)
    rng = random.Random(15)
    r = rng.randrange(1, p)
    Ar = np.array([[O.poly_eval(Ah[i, l], r, p) for l in range(N)] for i in range(N)], dtype=object)
    Br = np.array([[O.poly_eval(Bh[l, j], r, p) for j in range(N)] for l in range(N)], dtype=object)
    ref = (Ar @ Br) % p
    for i in range(0, N, 5):
        for j in range(N):
            assert O.poly_eval(C[i, j], r, p) == ref[i, j], (i, j)
    # one entry in full: sum of 32 oracle products (the oracle's NTT product, pinned)
    acc = np.zeros(2 * d - 1, dtype=np.uint64)
    for l in range(N):
        acc = O.vec_addmod(acc, O.poly_mul_ntt(Ah[0, l], Bh[l, 0], p, g), p)
    assert np.array_equal(u64(C[0, 0]), acc)


# ------------------------------------------------------------------ int_mul
def _to_int(limbs):
    return int.from_bytes(np.asarray(limbs, dtype="<u2").tobytes(), "little")


def _to_int32(limbs):
    return int.from_bytes(np.asarray(limbs, dtype="<u4").tobytes(), "little")


def _limbs32(seed, n):
    return (limbs16(seed, 1, 2 * n).view(np.uint32)).copy()


@pytest.mark.parametrize("na,nb", [(1, 1), (2, 2), (3, 1), (300, 257), (2048, 2049), (4096, 4096), (5000, 3),
                                   (10000, 12345), (1 << 15, 1 << 15), (40000, 70000)])
def test_int_mul_u32_three_prime(mm, O, na, nb):
    # P:971-979 three-prime FFT product vs Python big integers (library routine)
    a, b = _limbs32(na, na), _limbs32(nb + 1, nb)
    c = host(mm.int_mul_u32(dev(a), dev(b)))
    assert c.dtype == np.uint32 and c.size == na + nb
    assert _to_int32(c) == _to_int32(a) * _to_int32(b)


@pytest.mark.parametrize("m,kk,n,na,nb", [(2, 2, 2, 3, 3), (3, 4, 2, 100, 50), (1, 1, 1, 1, 1), (2, 3, 4, 2000, 3000)])
def test_int_matmul_u32(mm, O, m, kk, n, na, nb):
    # P:981-989 vs Python integers: C_ij = sum_l A_il B_lj
    A = np.stack([_limbs32(1000 * i + na, na) for i in range(m * kk)]).reshape(m, kk, na)
    B = np.stack([_limbs32(2000 * i + nb, nb) for i in range(kk * n)]).reshape(kk, n, nb)
    C = host(mm.int_matmul_u32(dev(A), dev(B)))
    for i in range(m):
        for j in range(n):
            ref = sum(_to_int32(A[i, l]) * _to_int32(B[l, j]) for l in range(kk))
            assert _to_int32(C[i, j]) == ref, (i, j)
    # all limbs 0xFFFFFFFF: every coefficient at kk min(na,nb) (2^32-1)^2
    A = np.full((m, kk, na), 0xFFFFFFFF, dtype=np.uint32)
    B = np.full((kk, n, nb), 0xFFFFFFFF, dtype=np.uint32)
    C = host(mm.int_matmul_u32(dev(A), dev(B)))
    ref = kk * ((1 << (32 * na)) - 1) * ((1 << (32 * nb)) - 1)
    assert all(_to_int32(C[i, j]) == ref for i in range(m) for j in range(n))


@pytest.mark.parametrize("N", [1, 2, 4097, 1 << 16, 1 << 20])
def test_int_mul_u32_all_ones(mm, O, N):
    # (2^(32N) - 1)^2: every coefficient at its maximum N (2^32 - 1)^2 (closed form);
    # N = 2^20: Table 16's size, raw limbs reduced in the TMA column loader
    a = np.full(N, 0xFFFFFFFF, dtype=np.uint32)
    c = host(mm.int_mul_u32(dev(a), dev(a)))
    ref = np.zeros(2 * N, dtype=np.uint32)
    ref[0] = 1
    ref[N] = 0xFFFFFFFE
    ref[N + 1:] = 0xFFFFFFFF
    assert np.array_equal(c, ref)


def test_int_mul_u32_paper_max(mm, O):
    # Table 16's largest size: 32 x 2^20-bit operands (na = nb = 2^20, transform 2^21);
    # checked by casting out random 61-bit primes and on the low 2^11 limbs exactly
    n = 1 << 20
    a, b = _limbs32(71, n), _limbs32(72, n)
    c = host(mm.int_mul_u32(dev(a), dev(b)))
    rng = random.Random(20)
    for _ in range(3):
        q = rng.randrange(1 << 60, 1 << 61) | 1
        assert O.limbs_mod(c.view(np.uint16), q) == O.limbs_mod(a.view(np.uint16), q) * O.limbs_mod(b.view(np.uint16), q) % q
    k = 1 << 11
    lo = _to_int32(a[:k]) * _to_int32(b[:k]) % (1 << (32 * k))
    assert _to_int32(c[:k]) == lo
    # and the same product through the Goldilocks path (16-bit limbs)
    c16 = host(mm.int_mul_u16(dev(a.view(np.uint16)), dev(b.view(np.uint16))))
    assert np.array_equal(c16.view(np.uint32), c)


@pytest.mark.parametrize("na,nb", [(1, 1), (2, 2), (3, 1), (300, 257), (2048, 2049), (4096, 4096),
                                   (5000, 3), (10000, 12345)])
def test_int_mul_random(mm, O, na, nb):
    a, b = limbs16(na, 1, na), limbs16(nb, 2, nb)
    c = host(mm.int_mul_u16(dev(a), dev(b)))
    assert _to_int(c) == _to_int(a) * _to_int(b)
    if na * nb <= 1 << 24:
        assert np.array_equal(c, O.int_mul_schoolbook_u16(a, b))


@pytest.mark.parametrize("N", [1, 2, 4095, 4097, 1 << 16, 1 << 20, 3 << 20])
def test_int_mul_all_ffff(mm, O, N):
    # (2^(16N) - 1)^2 = [1, 0 x (N-1), 0xFFFE, 0xFFFF x (N-1)]: max carries & coefficients
    a = np.full(N, 0xFFFF, dtype=np.uint16)
    c = host(mm.int_mul_u16(dev(a), dev(a)))
    expect = np.array([1] + [0] * (N - 1) + [0xFFFE] + [0xFFFF] * (N - 1), dtype=np.uint16)
    assert np.array_equal(c, expect)


def test_int_mul_medium_vs_oracle(mm, O):
    n = 1 << 18
    a, b = limbs16(7, 1, n), limbs16(7, 2, n)
    c = host(mm.int_mul_u16(dev(a), dev(b)))
    assert np.array_equal(c, O.int_mul_ntt_u16(a, b))


@pytest.fixture(scope="module")
def c5_ref(O):
    """BASELINE C5 operands and the oracle's full product (P:973 with one prime,
    DESIGN R7): or_int_mul_ntt_u16 -- textbook NTTs of 2^25 with u128 %, then
    sequential carries (~1 min on one host core)."""
    n = 1 << 24
    a = limbs16(config_seed(5), 1, n)
    b = limbs16(config_seed(5), 2, n)
    return a, b, O.int_mul_ntt_u16(a, b)


@pytest.mark.slow
def test_int_mul_c5_full(mm, O, c5_ref):
    # BASELINE C5: two 2^28-bit integers (2^24 limbs) -> 2^25 limbs, every limb
    # against the oracle product, operands drawn on the device (bench launch config)
    n = 1 << 24
    ah, bh, ref = c5_ref
    a = gen.limbs16_torch(config_seed(5), 1, n, DEV).view(torch.uint16)
    b = gen.limbs16_torch(config_seed(5), 2, n, DEV).view(torch.uint16)
    assert np.array_equal(host(a), ah) and np.array_equal(host(b), bh)   # generator parity host/device
    c = host(mm.int_mul_u16(a, b))
    assert c.size == 2 * n
    assert np.array_equal(c, ref)
    # independent proxies of the oracle's own result (library / definition checks)
    K = 4096
    assert np.array_equal(ref[:K], O.int_mul_schoolbook_u16(ah[:K], bh[:K])[:K])
    for q in ((1 << 61) - 1, 2305843009213693921, 1152921504606846883):
        assert O.limbs_mod(ref, q) == O.mulmod(O.limbs_mod(ah, q), O.limbs_mod(bh, q), q)


@pytest.mark.slow
def test_int_mul_c5_all_ffff_full(mm, O):
    # C5's second case at full size: all-0xFFFF operands (maximal coefficients and
    # carry chains): (2^(16N) - 1)^2 = [1, 0 x (N-1), 0xFFFE, 0xFFFF x (N-1)]
    N = 1 << 24
    a = torch.full((N,), -1, dtype=torch.int16, device=DEV).view(torch.uint16)
    c = host(mm.int_mul_u16(a, a))
    expect = np.concatenate([np.array([1], dtype=np.uint16), np.zeros(N - 1, dtype=np.uint16),
                             np.array([0xFFFE], dtype=np.uint16), np.full(N - 1, 0xFFFF, dtype=np.uint16)])
    assert np.array_equal(c, expect)


# ------------------------------------------------------------------ four-step blocks
def _loopback_exchange(sends, G):
    """Equal-split all-to-all among G virtual ranks on one GPU."""
    chunk = sends[0].numel() // G
    return [torch.cat([sends[g][h * chunk:(h + 1) * chunk] for g in range(G)]) for h in range(G)]


@pytest.mark.parametrize("bits,p,g,k", [(32, P30, 3, 16), (64, PG, 7, 20), (32, P30, 3, 20)])
@pytest.mark.parametrize("G", [1, 2, 4, 8])
def test_fourstep_blocks_loopback(mm, O, bits, p, g, k, G):
    """The sharded transform of dist.py on one GPU: G virtual ranks, their
    column-block shards, a loopback all-to-all; every rank's row block equals
    its slice of the single-GPU transform, and the inverse restores the input."""
    from paper_1407_3383_b200.dist import ShardedNtt
    w = O.root_of_unity(g, k, p)
    plan = mm.NttPlan(bits, p, k, w, 1)
    x = residues(11, k, 1 << k, p)
    xt = dev(x)
    ref = plan.forward(xt, out=torch.empty_like(xt), order=mm.BITREV)
    sh = [ShardedNtt(plan, rank=r, world=G) for r in range(G)]
    n1 = sh[0].n1
    xv = xt.view(torch.int64 if bits == 64 else torch.int32).reshape(-1, n1)
    blocks = [xv[:, r * sh[0].c1:(r + 1) * sh[0].c1].contiguous().view(xt.dtype) for r in range(G)]
    recv = _loopback_exchange([sh[r].forward_cols(blocks[r]) for r in range(G)], G)
    rows = [sh[h].forward_rows(recv[h]) for h in range(G)]
    got = torch.cat(rows, dim=0).reshape(-1)
    assert torch.equal(got.view(torch.int64 if bits == 64 else torch.int32),
                       ref.view(torch.int64 if bits == 64 else torch.int32))
    recv2 = _loopback_exchange([sh[h].inverse_rows(rows[h]) for h in range(G)], G)
    back = [sh[r].inverse_cols(recv2[r]) for r in range(G)]
    for r in range(G):
        assert torch.equal(back[r].view(torch.int64 if bits == 64 else torch.int32),
                           blocks[r].view(torch.int64 if bits == 64 else torch.int32))


@pytest.mark.parametrize("bits,p,g,k", [(32, P30, 3, 16), (64, PG, 7, 20)])
@pytest.mark.parametrize("G", [1, 2, 4, 8])
def test_fourstep_p2p_scatter(mm, O, bits, p, g, k, G):
    """Fused column pass + transpose (mm_ntt_fwd_cols_p2p): G virtual ranks on one
    GPU scatter their rows straight into each other's receive buffers; the
    row pass on those buffers equals the single-GPU transform."""
    from paper_1407_3383_b200.dist import ShardedNtt
    w = O.root_of_unity(g, k, p)
    plan = mm.NttPlan(bits, p, k, w, 1)
    x = residues(13, k, 1 << k, p)
    xt = dev(x)
    ref = plan.forward(xt, out=torch.empty_like(xt), order=mm.BITREV)
    sh = [ShardedNtt(plan, rank=r, world=G) for r in range(G)]
    n1, c1 = sh[0].n1, sh[0].c1
    sv = torch.int64 if bits == 64 else torch.int32
    xv = xt.view(sv).reshape(-1, n1)
    blocks = [xv[:, r * c1:(r + 1) * c1].contiguous().view(xt.dtype) for r in range(G)]
    recv = [torch.full_like(sh[r].forward_cols(blocks[r]), 0) for r in range(G)]
    ptrs = [t.data_ptr() for t in recv]
    for r in range(G):
        sh[r].forward_p2p(blocks[r], recv[r], ptrs)
    rows = [sh[h].forward_rows(recv[h]) for h in range(G)]
    got = torch.cat([t.view(sv) for t in rows], dim=0).reshape(-1)
    assert torch.equal(got, ref.view(sv))
    # and equal to the NCCL-style path (loopback all-to-all of forward_cols)
    recv2 = _loopback_exchange([sh[r].forward_cols(blocks[r]).view(sv) for r in range(G)], G)
    for h in range(G):
        assert torch.equal(recv[h].view(sv), recv2[h])


def _loopback_int_mul(mm, a, b, k, G):
    """dist.ShardedIntMul on one GPU: G virtual ranks, loopback all-to-alls, ring
    and all-gather; returns the product limbs reassembled in natural order."""
    from paper_1407_3383_b200.dist import ShardedIntMul
    p = PG
    plan = mm.NttPlan(64, p, k, pow(7, (p - 1) >> k, p), 1)
    sh = [ShardedIntMul(plan, a.numel(), b.numel(), rank=r, world=G) for r in range(G)]
    i64 = torch.int64                                            # exchange signed views (cat on int64)
    ra = _loopback_exchange([s.forward_cols(a).view(i64) for s in sh], G)
    rb = _loopback_exchange([s.forward_cols(b).view(i64) for s in sh], G)
    rc = _loopback_exchange([sh[h].products(ra[h], rb[h]).view(i64) for h in range(G)], G)
    coef = [sh[r].coefficients(rc[r]) for r in range(G)]
    halo_out = [sh[r].carry_halo(coef[r]) for r in range(G)]
    halo_in = [halo_out[(r - 1) % G] for r in range(G)]          # ring: from rank r - 1
    agg_all = torch.cat([sh[r].carry_reduce(coef[r], halo_in[r]).view(torch.int32) for r in range(G)])
    agg_all = agg_all.view(torch.uint32)
    sh[0].carry_scan(agg_all)
    n2 = sh[0].nt.n2
    outs = [sh[r].carry_apply(coef[r], halo_in[r], agg_all[r * n2:(r + 1) * n2]) for r in range(G)]
    n = 1 << k
    full = torch.empty(n, dtype=torch.int16, device=DEV)
    for r in range(G):
        idx = sh[r].limb_indices().reshape(-1).to(DEV)
        full[idx] = outs[r].view(torch.int16).reshape(-1)
    return full.view(torch.uint16)[:a.numel() + b.numel()]


@pytest.mark.parametrize("G", [1, 2, 4, 8])
@pytest.mark.parametrize("na,nb,k", [(3000, 5000, 14), (1 << 15, 1 << 15, 17), (1 << 16, 100, 17)])
def test_sharded_int_mul_loopback(mm, O, na, nb, k, G):
    a, b = limbs16(na + 3, 1, na), limbs16(nb + 3, 2, nb)
    got = host(_loopback_int_mul(mm, dev(a), dev(b), k, G))
    assert _to_int(got) == _to_int(a) * _to_int(b)
    ones = np.full(na, 0xFFFF, dtype=np.uint16)                    # maximal carry chains
    got = host(_loopback_int_mul(mm, dev(ones), dev(ones), k, G))
    assert _to_int(got) == _to_int(ones) ** 2


@pytest.mark.slow
def test_sharded_int_mul_c5_loopback(mm, O, c5_ref):
    # BASELINE C5 shape: 2^24 x 2^24 limbs, n = 2^25 (2^12-point column tiles, k = 25
    # tables), 8 virtual ranks; every limb equal to the oracle product
    n = 1 << 24
    a = gen.limbs16_torch(config_seed(5), 1, n, DEV).view(torch.uint16)
    b = gen.limbs16_torch(config_seed(5), 2, n, DEV).view(torch.uint16)
    for G in (2, 8):
        got = host(_loopback_int_mul(mm, a, b, 25, G))
        assert np.array_equal(got, c5_ref[2]), G


@pytest.mark.parametrize("bits,p,g,k", [(32, P30, 3, 16), (64, PG, 7, 20), (64, PG, 7, 24)])
def test_dist_c_abi_single_rank(mm, O, bits, p, g, k):
    # mm_dist_create / mm_ntt_forward_dist / mm_ntt_inverse_dist through the C ABI
    # with a one-rank NCCL communicator, then the peer-memory transport (device
    # flags, alternating receive buffers: epochs 1-3 cover the free-flag wait)
    w = O.root_of_unity(g, k, p)
    plan = mm.NttPlan(bits, p, k, w, 1)
    inf = plan.info()
    assert (inf["word_bits"], inf["batch"], inf["passes"]) == (bits, 1, 2)
    x = residues(21, k, 1 << k, p)
    xt = dev(x).reshape(inf["n2"], inf["n1"])
    ref = host(plan.forward(xt.reshape(-1), out=torch.empty_like(xt.reshape(-1)), order=mm.BITREV))
    if k <= 20:
        assert np.array_equal(u64(ref), O.to_bitrev(O.ntt(x, w, p)))
    D = mm.Dist.single()
    assert D.info()["world"] == 1 and D.info()["nccl_version"] > 0
    y = D.ntt_forward(plan, xt)
    assert np.array_equal(host(y).reshape(-1), ref)
    assert np.array_equal(host(D.ntt_inverse(plan, y)).reshape(-1), x)
    D.enable_p2p(xt.numel() * xt.element_size())
    assert D.info()["p2p_bytes"] >= xt.numel() * xt.element_size()
    for e in range(3):
        y = D.ntt_forward(plan, xt)
        assert np.array_equal(host(y).reshape(-1), ref), e
    assert D.p2p_status() == 0
    D.close()


@pytest.mark.parametrize("na,nb", [(3000, 5000), (1 << 15, 1 << 15), (1 << 16, 100)])
def test_dist_int_mul_c_abi_single_rank(mm, O, na, nb):
    # mm_int_mul_u16_dist with one rank: the [n2][c1] block is the whole product
    D = mm.Dist.single()
    a, b = limbs16(na + 5, 1, na), limbs16(nb + 5, 2, nb)
    L = D.int_mul_layout(na, nb)
    assert L["c1"] == L["n1"] and L["n1"] * L["n2"] == 1 << L["log2n"]
    got = host(D.int_mul_u16(dev(a), dev(b))).reshape(-1)
    assert np.array_equal(got[:na + nb], O.int_mul_ntt_u16(a, b))
    assert not got[na + nb:].any()
    D.close()


@pytest.mark.slow
def test_dist_int_mul_c_abi_c5_full(mm, O, c5_ref):
    # mm_int_mul_u16_dist (one-rank communicator) at the full C5 shape, every
    # limb against the oracle's product
    n = 1 << 24
    a = gen.limbs16_torch(config_seed(5), 1, n, DEV).view(torch.uint16)
    b = gen.limbs16_torch(config_seed(5), 2, n, DEV).view(torch.uint16)
    D = mm.Dist.single()
    got = host(D.int_mul_u16(a, b)).reshape(-1)
    D.close()
    assert np.array_equal(got[:2 * n], c5_ref[2])


def test_ntt_natural_order_stream_temporaries(mm, O):
    # NATURAL-order four-step calls permute through library-pool temporaries:
    # repeated calls on two streams sharing one plan stay correct
    p, k, B = P30, 16, 64
    w = O.root_of_unity(3, k, p)
    plan = mm.NttPlan(32, p, k, w, B)
    x = gen.residues_torch(config_seed(3), 9, B << k, p, DEV).view(torch.uint32)
    ref = plan.forward(x, out=torch.empty_like(x), order=mm.NATURAL)
    s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
    outs = []
    for s in (s1, s2, s1, s2):
        s.wait_stream(torch.cuda.current_stream())
        with torch.cuda.stream(s):
            outs.append(plan.forward(x, out=torch.empty_like(x), order=mm.NATURAL))
    torch.cuda.synchronize()
    for o in outs:
        assert torch.equal(o.view(torch.int32), ref.view(torch.int32))
    assert np.array_equal(u64(host(ref[:1 << k])), O.ntt(host(x[:1 << k]), w, p))


def _ipc_worker(rank, world, port):
    import os
    import torch.distributed as dist
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import ctypes
        import paper_1407_3383_b200 as m
        from paper_1407_3383_b200.dist import close_peer_pointers, peer_pointers
        torch.cuda.set_device(0)
        big = torch.zeros(4096 + 1024, dtype=torch.int32, device="cuda")
        # buffers at nonzero offsets inside their allocations (a caching
        # allocator's usual placement): 16 KiB + 4 KiB per rank in
        buf = big[4096 + 1024 * 0:][:1024] if rank == 0 else big[4096 - 1024:][:1024]
        assert m.ipc_handle(buf)[1] > 0
        ptrs, bases = peer_pointers(buf)
        # each rank writes its id into its slot of every peer's buffer through the opened pointers
        for h, q in enumerate(ptrs):
            src = torch.full((4,), rank + 1, dtype=torch.int32, device="cuda")
            torch.cuda.synchronize()
            ctypes.CDLL("libcudart.so").cudaMemcpy(ctypes.c_void_p(q + 16 * rank), ctypes.c_void_p(src.data_ptr()),
                                                   ctypes.c_size_t(16), 3)
        torch.cuda.synchronize()
        dist.barrier()
        got = buf[:4 * world].view(world, 4).cpu()
        assert all((got[r] == r + 1).all() for r in range(world)), got
        dist.barrier()
        close_peer_pointers(bases)
    finally:
        dist.destroy_process_group()


def test_ipc_peer_pointers(mm):
    # CUDA IPC plumbing of the peer-scatter path: two processes on one GPU
    # exchange handles (gloo) and write into each other's buffers
    import socket
    import torch.multiprocessing as mp
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    mp.spawn(_ipc_worker, args=(2, port), nprocs=2, join=True)


def test_debug_range_checks(mm, O, monkeypatch):
    # MMNTT_DEBUG=1: non-canonical residues are refused with MM_E_RANGE (header
    # conventions) by the NTT, product and numeric entry points; canonical ones pass
    monkeypatch.setenv("MMNTT_DEBUG", "1")
    for bits, p, g, k in [(32, P30, 3, 10), (32, P30, 3, 16), (64, PG, 7, 12), (64, PG, 7, 20)]:
        w = O.root_of_unity(g, k, p)
        plan = mm.NttPlan(bits, p, k, w, 2)
        x = residues(3, k, 2 << k, p)
        xt = dev(x)
        plan.forward(xt.clone(), order=mm.BITREV)                       # in range: fine
        bad = xt.clone()
        bad.view(torch.int64 if bits == 64 else torch.int32)[(1 << k) + 5] = -1   # 2^32 - 1 / 2^64 - 1 >= p
        for fn in (plan.forward, plan.inverse):
            with pytest.raises(mm.MMError) as e:
                fn(bad.clone(), order=mm.BITREV)
            assert e.value.status == 5
    a = dev(residues(4, 1, 3 * 700, P30).reshape(3, 700))
    b = dev(residues(4, 2, 3 * 900, P30).reshape(3, 900))
    mm.poly_mul(a, b, P30, 3)
    a.view(torch.int32)[2, 699] = P30
    with pytest.raises(mm.MMError):
        mm.poly_mul(a, b, P30, 3)
    with pytest.raises(mm.MMError):
        mm.poly_mul_tft(a.repeat(1, 30), b.repeat(1, 30), P30, 3)
    M = mm.ModNum(64, 65537)
    xf = torch.tensor([1.0, 2.5, 3.0, 4.0], dtype=torch.float64, device=DEV)   # 2.5 is not an integer
    with pytest.raises(mm.MMError):
        M.mul(xf, xf)
    monkeypatch.delenv("MMNTT_DEBUG")
    mm.poly_mul(a, b, P30, 3)                                             # trusted again


def test_release_cached(mm, O):
    # mm_release_cached frees the cached plans / workspaces; later calls rebuild them
    a = residues(8, 1, 2 * 5000, P30).reshape(2, 5000)
    b = residues(8, 2, 2 * 3000, P30).reshape(2, 3000)
    c1 = host(mm.poly_mul(dev(a), dev(b), P30, 3))
    ia, ib = limbs16(8, 3, 20000), limbs16(8, 4, 30000)
    i1 = host(mm.int_mul_u16(dev(ia), dev(ib)))
    mm.release_cached()
    assert np.array_equal(host(mm.poly_mul(dev(a), dev(b), P30, 3)), c1)
    assert np.array_equal(host(mm.int_mul_u16(dev(ia), dev(ib))), i1)
    assert np.array_equal(u64(c1[1]), O.poly_mul_ntt(a[1], b[1], P30, 3))


def test_poly_mul_fork_streams(mm, O):
    # C3 shape, 512 products: the sub-batch fork (mm_set_product_streams 2 and 3)
    # equals the one-stream result and the oracle, also inside a CUDA graph
    p, g, B, d = P30, 3, 512, 1 << 15
    a = gen.residues_torch(config_seed(3), 7, B * d, p, DEV).view(torch.uint32).reshape(B, d)
    b = gen.residues_torch(config_seed(3), 8, B * d, p, DEV).view(torch.uint32).reshape(B, d)
    mm.set_product_streams(1)
    ref = mm.poly_mul(a, b, p, g)
    try:
        for ns in (2, 3):
            mm.set_product_streams(ns)
            c = mm.poly_mul(a, b, p, g)
            assert torch.equal(c.view(torch.int32), ref.view(torch.int32)), ns
        mm.set_product_streams(2)
        c = torch.zeros_like(ref)
        s = torch.cuda.Stream()
        s.wait_stream(torch.cuda.current_stream())
        graph = torch.cuda.CUDAGraph()
        with torch.cuda.stream(s):
            mm.poly_mul(a, b, p, g, out=c)                       # warm (plans, workspaces)
            with torch.cuda.graph(graph, stream=s):
                mm.poly_mul(a, b, p, g, out=c)
        torch.cuda.synchronize()
        c.zero_()
        graph.replay()
        torch.cuda.synchronize()
        assert torch.equal(c.view(torch.int32), ref.view(torch.int32))
        for r in (0, 255, 256, 511):                              # both halves of the fork
            assert np.array_equal(u64(host(ref[r])), O.poly_mul_ntt(host(a[r]), host(b[r]), p, g)), r
        with pytest.raises(mm.MMError):
            mm.set_product_streams(0)
    finally:
        mm.set_product_streams(2)


def test_poly_mul_fork_odd_batch_strided(mm, O):
    # 257 products (sub-batches of 129 + 128) with padded output rows (ldc = 2^16):
    # the fork path equals the one-stream path, sampled rows equal the oracle
    p, g, B, d = P30, 3, 257, (1 << 15) - 3
    a = gen.residues_torch(config_seed(3), 11, B * d, p, DEV).view(torch.uint32).reshape(B, d)
    b = gen.residues_torch(config_seed(3), 12, B * d, p, DEV).view(torch.uint32).reshape(B, d)
    cp = torch.zeros((B, 1 << 16), dtype=torch.uint32, device=DEV)
    c = cp[:, :2 * d - 1]
    mm.set_product_streams(2)
    mm.poly_mul(a, b, p, g, out=c)
    mm.set_product_streams(1)
    try:
        ref = mm.poly_mul(a, b, p, g)
    finally:
        mm.set_product_streams(2)
    assert torch.equal(c.contiguous().view(torch.int32), ref.view(torch.int32))
    assert not cp[:, 2 * d - 1:].view(torch.int32).any()          # padding columns untouched
    for r in (0, 128, 129, 256):
        assert np.array_equal(u64(host(ref[r])), O.poly_mul_ntt(host(a[r]), host(b[r]), p, g)), r


@pytest.mark.parametrize("batch", [1, 3])
def test_ntt16_natural_in_place(mm, O, batch):
    # the natural-order 2^16 row passes, in place and out of place, batch 1 and 3
    p, k = P30, 16
    w = O.root_of_unity(3, k, p)
    plan = mm.NttPlan(32, p, k, w, batch)
    x = residues(17, batch, batch << k, p).reshape(batch, 1 << k)
    xt = dev(x)
    y = xt.clone()
    plan.forward(y, order=mm.NATURAL)                                 # in place
    nat = O.ntt_rows(x, w, p)
    assert np.array_equal(u64(host(y)), nat)
    z = plan.inverse(y, out=torch.empty_like(y), order=mm.NATURAL)
    assert torch.equal(z, xt)
    plan.inverse(y, order=mm.NATURAL)                                 # in place
    assert torch.equal(y, xt)


# ------------------------------------------------------------------ mm_run_jobs (one launch)
def test_jobs_c1_one_launch(mm, O):
    # BASELINE C1 as ONE launch: 16 round trips of 2^10 (forward spectrum in
    # natural order kept) and the 512 x 512 product, against the oracle
    p, k = P30, 10
    w = O.root_of_unity(3, k, p)
    x = residues(config_seed(1), 1, 16 << k, p).reshape(16, 1 << k)
    a = residues(config_seed(1), 2, 512, p)
    b = residues(config_seed(1), 3, 512, p)
    plan = mm.NttPlan(32, p, k, w, 16)
    xt = dev(x)
    y, z = torch.empty_like(xt), torch.empty_like(xt)
    c = torch.empty(1023, dtype=torch.uint32, device=DEV)
    jb = mm.Jobs()
    for r in range(16):
        jb.roundtrip(plan, xt[r], z[r], out=y[r], order=mm.NATURAL)
    jb.poly_mul(dev(a), dev(b), p, 3, c)
    jb.run()                      # the first call may build the product's cached plan (table kernels)
    n0 = mm.lib().mm_launch_count()
    jb.run()
    assert mm.lib().mm_launch_count() - n0 == 1
    assert np.array_equal(u64(host(y)), O.ntt_rows(x, w, p))
    assert np.array_equal(host(z), x)
    assert np.array_equal(u64(host(c)), O.poly_mul_schoolbook(a, b, p))


@pytest.mark.parametrize("p,g", [(P30, 3), (469762049, 3), (7681, 17)])
def test_jobs_mixed_sizes(mm, O, p, g):
    # every size 2^1 .. 2^12, forward and inverse in both orders, round trips,
    # ragged products -- all in one call
    rng = random.Random(p)
    jb, checks = mm.Jobs(), []
    for k in range(1, 13):
        if (p - 1) % (1 << k):
            continue
        w = O.root_of_unity(g, k, p)
        plan = mm.NttPlan(32, p, k, w, 1)
        x = residues(rng.randrange(1 << 30), 1, 1 << k, p)
        for order in (mm.NATURAL, mm.BITREV):
            ref = O.ntt(u64(x), w, p)
            ref = ref if order == mm.NATURAL else O.to_bitrev(ref)
            yf = torch.empty(1 << k, dtype=torch.uint32, device=DEV)
            jb.forward(plan, dev(x), yf, order=order)
            checks.append((yf, ref))
            yi = torch.empty_like(yf)
            jb.inverse(plan, dev(ref.astype(np.uint32)), yi, order=order)
            checks.append((yi, u64(x)))
        yr = torch.empty(1 << k, dtype=torch.uint32, device=DEV)
        jb.roundtrip(plan, dev(x), yr)
        checks.append((yr, u64(x)))
    for la, lb in [(1, 1), (1, 9), (3, 2), (100, 29), (513, 511), (2048, 2049), (4000, 97)]:
        if (p - 1) % (1 << max(1, (la + lb - 2).bit_length())):
            continue
        a = residues(rng.randrange(1 << 30), 2, la, p)
        b = residues(rng.randrange(1 << 30), 3, lb, p)
        c = torch.empty(la + lb - 1, dtype=torch.uint32, device=DEV)
        jb.poly_mul(dev(a), dev(b), p, g, c)
        checks.append((c, O.poly_mul_schoolbook(a, b, p)))
    jb.run()
    for t, ref in checks:
        assert np.array_equal(u64(host(t)), ref)


def test_jobs_many_and_errors(mm, O):
    # 600 jobs: a 256-job launch, another, then an 88-job one
    p, k = P30, 6
    w = O.root_of_unity(3, k, p)
    plan = mm.NttPlan(32, p, k, w, 1)
    x = residues(config_seed(1), 9, 600 << k, p).reshape(600, 1 << k)
    xt = dev(x)
    y = torch.empty_like(xt)
    jb = mm.Jobs()
    for r in range(600):
        jb.forward(plan, xt[r], y[r], order=mm.BITREV)
    jb.run()
    n0 = mm.lib().mm_launch_count()
    jb.run()
    assert mm.lib().mm_launch_count() - n0 == 3
    yh = u64(host(y))
    for r in range(0, 600, 37):
        assert np.array_equal(yh[r], O.to_bitrev(O.ntt(u64(x[r]), w, p)))
    # a job outside the scope fails the whole call before anything launches
    big = mm.NttPlan(32, p, 14, O.root_of_unity(3, 14, p), 1)
    xb = torch.zeros(1 << 14, dtype=torch.uint32, device=DEV)
    bad = mm.Jobs().forward(plan, xt[0], y[0]).forward(big, xb, torch.empty_like(xb))
    n0 = mm.lib().mm_launch_count()
    with pytest.raises(mm.MMError):
        bad.run()
    assert mm.lib().mm_launch_count() == n0
    with pytest.raises(mm.MMError):
        mm.Jobs().poly_mul(dev(x[0]), dev(x[1]), 1000003, 2, torch.empty(127, dtype=torch.uint32, device=DEV)).run()


def test_gold_tma_and_plain_kernels_agree(mm, O):
    # The TMA-staged Goldilocks passes (column tiles, bulk-copied rows) and the
    # per-thread-load kernels they replace (still used for sharded / segmented
    # / partial inputs) on the same C4-shaped transforms and a C5-shaped
    # product, each in a fresh process (MMNTT_GOLD_TMA is read once)
    import hashlib
    import subprocess
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    code = r"""
import hashlib, sys, torch
sys.path.insert(0, %r)
import gen, paper_1407_3383_b200 as mm
PG = (1 << 64) - (1 << 32) + 1
dev = torch.device("cuda")
x = gen.residues_torch(gen.config_seed(4), 21, 2 << 24, PG, dev).view(torch.uint64)
plan = mm.NttPlan(64, PG, 24, pow(7, (PG - 1) >> 24, PG), 2)
y = plan.forward(x, out=torch.empty_like(x), order=mm.BITREV)
z = plan.inverse(y, out=torch.empty_like(y), order=mm.BITREV)
a = gen.limbs16_torch(gen.config_seed(5), 21, 1 << 24, dev).view(torch.uint16)
b = gen.limbs16_torch(gen.config_seed(5), 22, 1 << 24, dev).view(torch.uint16)
c = mm.int_mul_u16(a, b)
h = hashlib.sha256()
for t in (y, z, c):
    h.update(t.cpu().numpy().tobytes())
print(h.hexdigest(), bool(torch.equal(z, x)))
""" % root
    outs = []
    for v, fused in (("1", None), ("0", None), ("1", "1")):   # the last: the single-pass look-back carry
        env = dict(os.environ, MMNTT_GOLD_TMA=v)
        if fused:
            env["MMNTT_CARRY_FUSED"] = fused
        r = subprocess.run([sys.executable, "-c", code], env=env, capture_output=True, text=True, timeout=600)
        assert r.returncode == 0, r.stderr[-2000:]
        outs.append(r.stdout.split()[-2:])
    assert all(o[1] == "True" for o in outs)
    assert outs[0][0] == outs[1][0] == outs[2][0]


@pytest.mark.parametrize("cfg", ["c1", "c2"])
def test_bench_config_line(cfg):
    # bench.py --config: one contract line for that BASELINE config, with the
    # library's kernels counted inside the timed region
    import json
    import subprocess
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    r = subprocess.run([sys.executable, "bench.py", "--config", cfg, "--steps", "3", "--warmup", "3",
                        "--no-cpu-baseline"], cwd=root, capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stderr[-2000:]
    line = json.loads(r.stdout.strip().splitlines()[-1])
    assert line["config"]["config"] == cfg.upper() and line["value"] > 0 and line["gpu_launches"] >= 3
    assert line["roofline"]["frac"] > 0 and line["e2e"]["h2d_bytes_per_step"] > 0
    assert line["clocks"]["sm_mhz"] is None or line["clocks"]["sm_mhz"] > 0
