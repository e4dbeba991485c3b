"""Multi-GPU plumbing: one length-n transform split across ranks (Algorithm 1).

Algorithm 1 with l = n views the input as n2 rows x n1 columns
(a[j2 n1 + j1]).  Steps 1-2 (column TFFTs + twiddle w^(j1 [i2])) touch one
column at a time, steps 3-4 (row TFFTs) one row at a time, so the transform
shards by columns for the first half and by rows for the second, with one
all-to-all in between -- the "cache-friendly transposition" of P:925 becomes
an NCCL all-to-all over NVLink.

Layouts (rank g of G, c1 = n1 / G, r2 = n2 / G):
  * input  : column block [n2][c1] holding columns [g c1, (g+1) c1) of the
             natural-order input (what rank g draws from the generator);
  * output : row block [r2][n1] holding positions [g r2 n1, (g+1) r2 n1) of
             the bit-mirrored (TFT) output, i.e. rows i2 in
             [g r2, (g+1) r2) of Algorithm 1's step-4 layout;
  * inverse: the exact reverse (row block in, column block out, n^-1 applied).

Compute runs in libmmntt kernels (mm_ntt_fwd_cols / mm_ntt_fwd_rows_seg /
mm_ntt_inv_rows_seg / mm_ntt_inv_cols); torch.distributed (NCCL on GPUs,
gloo in the CPU tests) only moves bytes.  The row kernels read / write the
all-to-all buffers in place ("segmented rows"), so there is no reshuffle copy.
The `plan` argument only needs the four block methods and info(), which lets
the CPU tests drive the same orchestration with a reference backend.
"""
from __future__ import annotations

import torch
import torch.distributed as dist


def _bits(t: torch.Tensor) -> torch.Tensor:
    """Signed view of the same bytes (collectives are defined on signed ints)."""
    return t.view(torch.int64 if t.element_size() == 8 else torch.int32)


class ShardedNtt:
    """A single transform of length n = n2 n1 sharded over the ranks of `group`."""

    def __init__(self, plan, group=None, rank=None, world=None):
        self.plan = plan
        self.group = group
        info = plan.info()
        self.n1, self.n2 = info["n1"], info["n2"]
        if info.get("passes", 2) != 2:
            raise ValueError("sharded transforms need a four-step plan (log2 n > 12)")
        # explicit (rank, world) without a process group: phases driven by the caller
        self.G = world if world is not None else dist.get_world_size(group)
        self.rank = rank if rank is not None else dist.get_rank(group)
        if self.n1 % self.G or self.n2 % self.G:
            raise ValueError(f"n1={self.n1}, n2={self.n2} must be divisible by world size {self.G}")
        self.c1, self.r2 = self.n1 // self.G, self.n2 // self.G

    # ---- forward: column block -> bit-mirrored row block
    def forward_cols(self, x_cols: torch.Tensor) -> torch.Tensor:
        """Steps 1-2 on my columns; returns the all-to-all send buffer (chunk h =
        rows [h r2, (h+1) r2) of my columns, for rank h)."""
        if tuple(x_cols.shape) != (self.n2, self.c1):
            raise ValueError(f"expected a [{self.n2}, {self.c1}] column block")
        y = torch.empty_like(x_cols)
        self.plan.fwd_cols(x_cols, y, self.rank * self.c1, self.c1)
        return y.reshape(-1)

    def forward_rows(self, recv: torch.Tensor) -> torch.Tensor:
        """Steps 3-4 on the receive buffer (G segments [r2][c1], segment g =
        columns [g c1, (g+1) c1)), read in place; returns my [r2][n1] row block."""
        out = torch.empty((self.r2, self.n1), dtype=recv.dtype, device=recv.device)
        self.plan.fwd_rows_seg(recv, out, self.rank * self.r2, self.r2, self.c1, self.r2 * self.c1)
        return out

    def forward_p2p(self, x_cols: torch.Tensor, recv: torch.Tensor, peer_ptrs) -> None:
        """Steps 1-2 with the transpose fused into the stores: rows of my
        column block go straight into the peers' receive buffers (peer_ptrs[h]
        = device address of rank h's `recv`, e.g. CUDA IPC-opened; recv is my
        own).  After every rank's call completes (a cross-rank barrier),
        forward_rows(recv) finishes the transform -- no all-to-all."""
        if tuple(x_cols.shape) != (self.n2, self.c1):
            raise ValueError(f"expected a [{self.n2}, {self.c1}] column block")
        self.plan.fwd_cols_p2p(x_cols, peer_ptrs, self.rank, self.rank * self.c1, self.c1)

    def forward(self, x_cols: torch.Tensor) -> torch.Tensor:
        send = self.forward_cols(x_cols)
        recv = torch.empty_like(send)
        dist.all_to_all_single(_bits(recv), _bits(send), group=self.group)
        return self.forward_rows(recv)

    # ---- inverse: bit-mirrored row block -> natural column block
    def inverse_rows(self, y_rows: torch.Tensor) -> torch.Tensor:
        """Inverse steps 4-3 + twiddle w^-(j1 [i2]); returns the send buffer
        (segment g = the columns of rank g)."""
        if tuple(y_rows.shape) != (self.r2, self.n1):
            raise ValueError(f"expected a [{self.r2}, {self.n1}] row block")
        send = torch.empty(self.G * self.r2 * self.c1, dtype=y_rows.dtype, device=y_rows.device)
        self.plan.inv_rows_seg(y_rows, send, self.rank * self.r2, self.r2, self.c1, self.r2 * self.c1)
        return send

    def inverse_cols(self, recv: torch.Tensor) -> torch.Tensor:
        """recv = [G][r2][c1] = rows 0..n2-1 of my columns: inverse steps 2-1, n^-1."""
        x = torch.empty((self.n2, self.c1), dtype=recv.dtype, device=recv.device)
        self.plan.inv_cols(recv.view(self.n2, self.c1), x, self.rank * self.c1, self.c1)
        return x

    def inverse(self, y_rows: torch.Tensor) -> torch.Tensor:
        send = self.inverse_rows(y_rows)
        recv = torch.empty_like(send)
        dist.all_to_all_single(_bits(recv), _bits(send), group=self.group)
        return self.inverse_cols(recv)

    # ---- index maps (used by tests and the bench to draw / check shards)
    def column_block_indices(self) -> torch.Tensor:
        """Natural input indices j2 n1 + j1 held by this rank, as [n2][c1]."""
        j2 = torch.arange(self.n2).view(-1, 1)
        j1 = torch.arange(self.rank * self.c1, (self.rank + 1) * self.c1).view(1, -1)
        return j2 * self.n1 + j1

    def row_block_positions(self) -> range:
        """Positions of the bit-mirrored output held by this rank."""
        return range(self.rank * self.r2 * self.n1, (self.rank + 1) * self.r2 * self.n1)


def peer_pointers(buf: torch.Tensor, group=None) -> tuple[list, list]:
    """Device addresses of every rank's `buf` as seen from this process (one
    node): (CUDA IPC handle, offset of buf inside its allocation) all-gathered,
    peers' allocations opened and the offsets added back (own rank: local).
    Returns (pointers, opened bases to pass to close_peer_pointers)."""
    import paper_1407_3383_b200 as mm
    G, g = dist.get_world_size(group), dist.get_rank(group)
    handles = [None] * G
    dist.all_gather_object(handles, mm.ipc_handle(buf), group=group)
    ptrs, bases = [], []
    for h in range(G):
        if h == g:
            ptrs.append(buf.data_ptr())
            continue
        base = mm.ipc_open(handles[h][0])
        bases.append(base)
        ptrs.append(base + handles[h][1])
    return ptrs, bases


def close_peer_pointers(bases) -> None:
    import paper_1407_3383_b200 as mm
    for b in bases:
        mm.ipc_close(b)


class ShardedIntMul:
    """One integer product a b sharded over the ranks of `group`.

    a, b: 16-bit little-endian limbs (every rank holds both: 2 B per limb), the
    product runs over p = 2^64 - 2^32 + 1 as in mm_int_mul_u16 (P:971-973 with
    one prime, R7).  Per rank: the column pass reads its columns of
    the zero-padded limb vectors in place (mm_ntt_fwd_cols_u16); one all-to-all
    per operand; one fused row kernel (steps 3-4 of both operands, pointwise
    product, inverse steps 4-3 and twiddle, mm_ntt_pmul_rows_seg); one
    all-to-all back; the inverse column pass (n^-1).  Rank g then holds the
    coefficients c_j, j = r n1 + g c1 + i, as n2 chunks of c1 consecutive j.
    Carries (evaluation at 2^16): each chunk needs the 4 coefficients before it
    (a ring send of [n2][4] words to the next rank), per-chunk (generate,
    propagate) pairs are all-gathered ([G][n2] words) and scanned in natural
    chunk order on every rank, then applied locally.  Output: the limbs of
    a b at the same positions, [n2][c1] 16-bit words (limb_indices()).

    `backend` supplies carry_chunks_{halo,reduce,scan,apply} (the library by
    default; the CPU tests pass a reference)."""

    def __init__(self, plan, na: int, nb: int, group=None, rank=None, world=None, backend=None):
        self.nt = ShardedNtt(plan, group, rank, world)
        self.plan, self.group = plan, group
        self.na, self.nb = na, nb
        self.nc, self.nout = na + nb - 1, na + nb
        n1, n2 = self.nt.n1, self.nt.n2
        if self.nout > n1 * n2:
            raise ValueError(f"na + nb = {self.nout} limbs exceed the transform length {n1 * n2}")
        if self.nt.c1 < 4:
            raise ValueError("column blocks must hold at least 4 columns (carry halo)")
        if backend is None:
            import paper_1407_3383_b200 as backend
        self.be = backend

    # ---- phases (each local; the collectives sit between them)
    def forward_cols(self, limbs: torch.Tensor) -> torch.Tensor:
        nt = self.nt
        y = torch.empty((nt.n2, nt.c1), dtype=torch.uint64, device=limbs.device)
        self.plan.fwd_cols_u16(limbs, y, nt.rank * nt.c1, nt.c1)
        return y.reshape(-1)

    def products(self, recv_a: torch.Tensor, recv_b: torch.Tensor) -> torch.Tensor:
        nt = self.nt
        send = torch.empty_like(recv_a)
        self.plan.pmul_rows_seg(recv_a, recv_b, send, nt.rank * nt.r2, nt.r2, nt.c1, nt.r2 * nt.c1)
        return send

    def coefficients(self, recv_c: torch.Tensor) -> torch.Tensor:
        return self.nt.inverse_cols(recv_c)

    def carry_halo(self, coef: torch.Tensor) -> torch.Tensor:
        halo = torch.empty((coef.shape[0], 4), dtype=coef.dtype, device=coef.device)
        return self.be.carry_chunks_halo(coef, halo)

    def carry_reduce(self, coef: torch.Tensor, halo_in: torch.Tensor) -> torch.Tensor:
        nt = self.nt
        agg = torch.empty(coef.shape[0], dtype=torch.uint32, device=coef.device)
        return self.be.carry_chunks_reduce(coef, halo_in, nt.n1, nt.rank * nt.c1, self.nc, self.nout,
                                           nt.rank == 0, agg)

    def carry_scan(self, agg_all: torch.Tensor) -> torch.Tensor:
        return self.be.carry_chunks_scan(agg_all, self.nt.G, self.nt.n2)

    def carry_apply(self, coef: torch.Tensor, halo_in: torch.Tensor, cin: torch.Tensor) -> torch.Tensor:
        nt = self.nt
        out = torch.empty(coef.shape, dtype=torch.uint16, device=coef.device)
        return self.be.carry_chunks_apply(coef, halo_in, nt.n1, nt.rank * nt.c1, self.nc, self.nout, nt.rank == 0,
                                          cin, out)

    # ---- collectives
    def _a2a(self, send: torch.Tensor) -> torch.Tensor:
        recv = torch.empty_like(send)
        dist.all_to_all_single(_bits(recv), _bits(send), group=self.group)
        return recv

    def _ring(self, halo_out: torch.Tensor) -> torch.Tensor:
        """halo_in = halo_out of rank g - 1 (rank 0 gets the last rank's)."""
        G, g = self.nt.G, self.nt.rank
        if G == 1:
            return halo_out.clone()
        halo_in = torch.empty_like(halo_out)
        grp = self.group
        nxt = dist.get_global_rank(grp, (g + 1) % G) if grp is not None else (g + 1) % G
        prv = dist.get_global_rank(grp, (g - 1) % G) if grp is not None else (g - 1) % G
        ops = [dist.P2POp(dist.isend, _bits(halo_out), nxt, grp), dist.P2POp(dist.irecv, _bits(halo_in), prv, grp)]
        for req in dist.batch_isend_irecv(ops):
            req.wait()
        return halo_in

    def __call__(self, a: torch.Tensor, b: torch.Tensor) -> torch.Tensor:
        if a.numel() != self.na or b.numel() != self.nb:
            raise ValueError("operand sizes differ from the plan")
        recv_a = self._a2a(self.forward_cols(a))
        recv_b = self._a2a(self.forward_cols(b))
        coef = self.coefficients(self._a2a(self.products(recv_a, recv_b)))
        halo_in = self._ring(self.carry_halo(coef))
        agg = self.carry_reduce(coef, halo_in)
        agg_all = torch.empty(self.nt.G * agg.numel(), dtype=agg.dtype, device=agg.device)
        dist.all_gather_into_tensor(_bits(agg_all), _bits(agg), group=self.group)
        self.carry_scan(agg_all)
        cin = agg_all[self.nt.rank * self.nt.n2:(self.nt.rank + 1) * self.nt.n2]
        return self.carry_apply(coef, halo_in, cin)

    def limb_indices(self) -> torch.Tensor:
        """Limb indices j of this rank's output block, as [n2][c1]."""
        return self.nt.column_block_indices()
