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
