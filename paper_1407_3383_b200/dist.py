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
