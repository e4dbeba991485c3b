"""Multi-rank orchestration of the sharded four-step transform on CPU (gloo).

The GPU kernels are replaced by a reference backend implementing the same
block semantics (column TFFT + twiddle, segmented row TFFT, and inverses)
from the oracle, so these tests pin the exchange logic of
paper_1407_3383_b200/dist.py -- column-block input, equal-split all-to-all,
segmented row blocks, bit-mirrored row-block output -- with real
torch.distributed collectives on world sizes 2 and 4.  The GPU loopback test
(test_gpu_parity.test_fourstep_blocks_loopback) pins the same layouts against
the kernels.
"""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import gen

P30 = 998244353
PG = (1 << 64) - (1 << 32) + 1


class RefPlan:
    """Oracle-backed stand-in for NttPlan's four-step block methods (test only)."""

    def __init__(self, p, g, k, k2):
        import oracle as O
        self.O, self.p, self.k, self.k2 = O, p, k, k2
        self.k1 = k - k2
        self.n1, self.n2 = 1 << self.k1, 1 << k2
        self.w = O.root_of_unity(g, k, p)
        self.winv = O.powmod(self.w, p - 2, p)

    def info(self):
        return {"n1": self.n1, "n2": self.n2, "passes": 2}

    def _np(self, t):
        return t.numpy().view(np.uint64).astype(np.uint64) if t.element_size() == 8 else \
            t.numpy().view(np.uint32).astype(np.uint64)

    def _put(self, out, arr):
        if out.element_size() == 8:
            out.copy_(torch.from_numpy(arr.astype(np.uint64).view(np.int64)).view(out.dtype).reshape(out.shape))
        else:
            out.copy_(torch.from_numpy(arr.astype(np.uint32).view(np.int32)).view(out.dtype).reshape(out.shape))

    def fwd_cols(self, x, out, col0, ncols):
        O, p = self.O, self.p
        X = self._np(x).reshape(self.n2, ncols)
        w2 = O.powmod(self.w, self.n1, p)
        Y = np.zeros_like(X)
        for c in range(ncols):
            col = O.to_bitrev(O.ntt(X[:, c], w2, p))          # step 1, bit-mirrored rows
            j1 = col0 + c
            tw = np.array([O.powmod(self.w, j1 * O.bitrev(t, self.k2), p) for t in range(self.n2)], dtype=np.uint64)
            Y[:, c] = O.vec_mulmod(col, tw, p)                 # step 2
        self._put(out, Y)

    def _gather(self, buf, nrows, seg_len, seg_stride):
        B = self._np(buf)
        rows = np.zeros((nrows, self.n1), dtype=np.uint64)
        for s in range(self.n1 // seg_len):
            seg = B[s * seg_stride: s * seg_stride + nrows * seg_len].reshape(nrows, seg_len)
            rows[:, s * seg_len:(s + 1) * seg_len] = seg
        return rows

    def fwd_rows_seg(self, recv, out, row0, nrows, seg_len, seg_stride):
        O, p = self.O, self.p
        rows = self._gather(recv, nrows, seg_len, seg_stride)
        w1 = O.powmod(self.w, self.n2, p)
        self._put(out, np.stack([O.to_bitrev(O.ntt(r, w1, p)) for r in rows]))   # steps 3-4

    def inv_rows_seg(self, y, send, row0, nrows, seg_len, seg_stride):
        O, p = self.O, self.p
        Y = self._np(y).reshape(nrows, self.n1)
        w1i = O.powmod(self.winv, self.n2, p)
        S = np.zeros(send.numel(), dtype=np.uint64)
        for r in range(nrows):
            i2 = row0 + r
            v = O.ntt(O.to_bitrev(Y[r]), w1i, p)              # unscaled inverse row TFFT
            tw = np.array([O.powmod(self.winv, j1 * O.bitrev(i2, self.k2), p) for j1 in range(self.n1)],
                          dtype=np.uint64)
            v = O.vec_mulmod(v, tw, p)
            for s in range(self.n1 // seg_len):
                S[s * seg_stride + r * seg_len: s * seg_stride + (r + 1) * seg_len] = v[s * seg_len:(s + 1) * seg_len]
        self._put(send, S)

    def inv_cols(self, x, out, col0, ncols):
        O, p = self.O, self.p
        X = self._np(x).reshape(self.n2, ncols)
        w2i = O.powmod(self.winv, self.n1, p)
        ninv = O.powmod(1 << self.k, p - 2, p)
        Y = np.zeros_like(X)
        for c in range(ncols):
            v = O.ntt(O.to_bitrev(X[:, c]), w2i, p)
            Y[:, c] = O.vec_mulmod(v, np.full(self.n2, ninv, dtype=np.uint64), p)
        self._put(out, Y)


    # ---- sharded integer product blocks (same semantics as the library's)
    def fwd_cols_u16(self, limbs, out, col0, ncols):
        L = limbs.numpy().view(np.uint16).astype(np.uint64)
        full = np.zeros(self.n1 * self.n2, dtype=np.uint64)
        full[:L.size] = L
        X = full.reshape(self.n2, self.n1)[:, col0:col0 + ncols].copy()
        self.fwd_cols(torch.from_numpy(X.view(np.int64)), out, col0, ncols)
        return out

    def pmul_rows_seg(self, a, b, out, row0, nrows, seg_len, seg_stride):
        O, p = self.O, self.p
        ta = torch.empty((nrows, self.n1), dtype=torch.int64)
        tb = torch.empty((nrows, self.n1), dtype=torch.int64)
        self.fwd_rows_seg(a, ta, row0, nrows, seg_len, seg_stride)
        self.fwd_rows_seg(b, tb, row0, nrows, seg_len, seg_stride)
        C = O.vec_mulmod(self._np(ta).reshape(-1), self._np(tb).reshape(-1), p).reshape(nrows, self.n1)
        self.inv_rows_seg(torch.from_numpy(C.astype(np.uint64).view(np.int64)), out, row0, nrows, seg_len,
                          seg_stride)
        return out


class RefCarry:
    """Reference for the chunked carry kernels: digits of c_j at 2^16, the
    (generate, propagate) chain, evaluated straight from the definitions."""

    @staticmethod
    def _coef(coef, halo, r, i, shift):
        if i >= 0:
            return int(coef[r, i])
        hr = r - 1 if shift else r
        return int(halo[hr, 4 + i]) if hr >= 0 else 0

    def _wg(self, coef, halo, n1, col0, nc, r, i, shift):
        def s_at(ii):
            jg = r * n1 + col0 + ii
            return sum((self._coef(coef, halo, r, ii - t, shift) >> (16 * t)) & 0xFFFF
                       for t in range(4) if 0 <= jg - t < nc)
        sj = s_at(i)
        sp = s_at(i - 1) if r * n1 + col0 + i > 0 else 0
        u = (sj & 0xFFFF) + (sp >> 16)
        return u & 0xFFFF, u >> 16

    @staticmethod
    def _u(t):
        return t.numpy().view(np.uint64) if t.element_size() == 8 else t.numpy().view(np.uint32)

    def carry_chunks_halo(self, coef, halo_out):
        C = self._u(coef)
        halo_out.copy_(torch.from_numpy(C[:, -4:].copy().view(np.int64)).view(halo_out.dtype))
        return halo_out

    def carry_chunks_reduce(self, coef, halo, n1, col0, nc, nout, shift, agg):
        C, H = self._u(coef), self._u(halo)
        res = []
        for r in range(C.shape[0]):
            G, P = 0, 1
            for i in range(C.shape[1]):
                if r * n1 + col0 + i >= nout:
                    continue
                w, g = self._wg(C, H, n1, col0, nc, r, i, shift)
                G, P = g | (int(w == 0xFFFF) & G), int(w == 0xFFFF) & P
            res.append(G | (P << 1))
        agg.copy_(torch.tensor(res, dtype=torch.int32).view(agg.dtype))
        return agg

    def carry_chunks_scan(self, agg_all, G, nrows):
        A = agg_all.numpy().view(np.uint32)
        carry, out = 0, A.copy()
        for q in range(G * nrows):
            at = (q % G) * nrows + q // G
            out[at] = carry
            gp = int(A[at])
            carry = (gp & 1) | ((gp >> 1) & carry)
        agg_all.copy_(torch.from_numpy(out.view(np.int32)).view(agg_all.dtype))
        return agg_all

    def carry_chunks_apply(self, coef, halo, n1, col0, nc, nout, shift, cin, out):
        C, H = self._u(coef), self._u(halo)
        Ci = cin.numpy().view(np.uint32)
        O = np.zeros(C.shape, dtype=np.uint16)
        for r in range(C.shape[0]):
            carry = int(Ci[r])
            for i in range(C.shape[1]):
                if r * n1 + col0 + i >= nout:
                    continue
                w, g = self._wg(C, H, n1, col0, nc, r, i, shift)
                O[r, i] = (w + carry) & 0xFFFF
                carry = g | (int(w == 0xFFFF) & carry)
        out.copy_(torch.from_numpy(O.view(np.int16)).view(out.dtype))
        return out


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _worker(rank, world, port, p, g, k, k2, dtype_bits):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import oracle as O
        from paper_1407_3383_b200.dist import ShardedNtt
        plan = RefPlan(p, g, k, k2)
        sh = ShardedNtt(plan)
        n = 1 << k
        full = gen.residues(21, k, n, p).astype(np.uint64)
        idx = sh.column_block_indices().numpy()
        block = full[idx]
        tdt = torch.int64 if dtype_bits == 64 else torch.int32
        ndt = np.int64 if dtype_bits == 64 else np.int32
        x = torch.from_numpy(block.astype(np.uint64 if dtype_bits == 64 else np.uint32).view(ndt)).to(tdt)
        y = sh.forward(x)
        ref = O.to_bitrev(O.ntt(full, O.root_of_unity(g, k, p), p))     # TFT order
        pos = sh.row_block_positions()
        got = y.numpy().view(np.uint64 if dtype_bits == 64 else np.uint32).astype(np.uint64).reshape(-1)
        assert np.array_equal(got, ref[pos.start:pos.stop]), f"rank {rank}: forward block mismatch"
        z = sh.inverse(y)
        back = z.numpy().view(np.uint64 if dtype_bits == 64 else np.uint32).astype(np.uint64)
        assert np.array_equal(back, block), f"rank {rank}: inverse mismatch"
        dist.barrier()
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 4])
@pytest.mark.parametrize("p,g,k,k2,bits", [(P30, 3, 8, 4, 32), (PG, 7, 9, 4, 64)])
def test_sharded_ntt_gloo(world, p, g, k, k2, bits):
    mp.spawn(_worker, args=(world, _free_port(), p, g, k, k2, bits), nprocs=world, join=True)


def _int_worker(rank, world, port, k, k2, na, nb, all_ones):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_1407_3383_b200.dist import ShardedIntMul
        plan = RefPlan(PG, 7, k, k2)
        sh = ShardedIntMul(plan, na, nb, backend=RefCarry())
        if all_ones:
            a = np.full(na, 0xFFFF, dtype=np.uint16)
            b = np.full(nb, 0xFFFF, dtype=np.uint16)
        else:
            a, b = gen.limbs16(31, 1, na), gen.limbs16(31, 2, nb)
        out = sh(torch.from_numpy(a.view(np.int16)), torch.from_numpy(b.view(np.int16)))
        prod = int.from_bytes(a.tobytes(), "little") * int.from_bytes(b.tobytes(), "little")
        ref = np.frombuffer(prod.to_bytes(2 * (na + nb), "little"), dtype=np.uint16)
        full = np.zeros(1 << k, dtype=np.uint16)
        full[:na + nb] = ref
        idx = sh.limb_indices().numpy()
        got = out.numpy().view(np.uint16)
        assert np.array_equal(got, full[idx]), f"rank {rank}: limb block mismatch"
        dist.barrier()
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 4])
@pytest.mark.parametrize("na,nb,ones", [(500, 400, False), (512, 512, True), (3, 700, False)])
def test_sharded_int_mul_gloo(world, na, nb, ones):
    # the sharded integer product with cross-rank carries
    mp.spawn(_int_worker, args=(world, _free_port(), 10, 4, na, nb, ones), nprocs=world, join=True)
