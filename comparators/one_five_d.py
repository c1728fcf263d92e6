"""NEXT-4 comparator: the 1.5D A-stationary SpMM the paper benchmarks against (§2;
baseline choice c = floor(sqrt(p)) at P:1212-1216).  A comparator, not the product: the local
products are cuSPARSE CSRMM through torch.sparse.mm, exactly as the paper's baseline used "the
same libraries and kernels", and the collectives are torch.distributed (NCCL on
GPUs, gloo in the CPU tests).  It never imports oracle/ and shares nothing with csrc/.

Layout.  p processors form a (p/c) x c grid; processor (i, j) has rank i*c + j.
  * A is cut into p tiles of (nc/p) x (n/c): row block i (X/Y tile i, rows [B_i, B_{i+1}) with
    B_t = floor(n t / (p/c))) times column block j, which is the union of the p/c^2 consecutive
    X tiles j*(p/c^2) .. (j+1)*(p/c^2) - 1.
  * X tile i is replicated on the c processors of grid row i; so is the result tile Y_i.
Step.
  * p/c^2 rounds; in round r the X tile t = j*(p/c^2) + r is broadcast within grid column j from
    its holder (t, j); every processor multiplies its (row block i) x (tile t) piece of A by it and
    accumulates into a partial Y_i.  Only one extra X tile is held at a time.
  * The c partial tiles of row block i are summed by an all-reduce.

Reading R24: P:321 says "each grid column performs an all-reduce"; the partial
tiles of one row block i live on the c processors of grid ROW i (they differ in their column
block j), so the all-reduce runs over the grid row.  The cost the paper states,
O(alpha p/c^2 log p + beta (nk/c + nkc/p)), is what this layout gives: nk/c received by
broadcasts (the n/c rows of a column block) plus an all-reduce of an nc/p x k tile.
c must divide p/c (c^2 | p); grid_c picks the largest such c <= floor(sqrt(p)).
"""
from __future__ import annotations

import math

import numpy as np


def grid_c(p: int) -> int:
    """Replication factor: floor(sqrt(p)), lowered until c^2 divides p (P:320's rounds)."""
    c = max(1, math.isqrt(p))
    while c > 1 and p % (c * c):
        c -= 1
    return c


def tile_bounds(n: int, q: int) -> list[int]:
    return [n * t // q for t in range(q + 1)]


def ledger(n: int, k: int, es: int, p: int, c: int, rank: int) -> dict:
    """Bytes rank receives per step under the layout above (broadcasts of the other tiles of its
    column block + a ring all-reduce of its Y tile), next to P:322's beta term nk/c + nkc/p."""
    q = p // c
    rounds = q // c
    B = tile_bounds(n, q)
    i, j = divmod(rank, c)
    bcast = sum((B[t + 1] - B[t]) for t in range(j * rounds, (j + 1) * rounds) if t != i) * k * es
    rows_i = B[i + 1] - B[i]
    allred = (2 * (c - 1) * rows_i * k * es) // c
    return {"c": c, "rounds": rounds, "bcast_recv_bytes": int(bcast), "allreduce_bytes": int(allred),
            "predicted_beta_bytes": int((n * k / c + n * k * c / p) * es)}


class OneFiveD:
    """1.5D A-stationary SpMM over a torch.distributed world (one rank per device)."""

    def __init__(self, n, row_ptr, col, val, k, torch_dtype, rank, world, device, c: int | None = None):
        import torch
        import torch.distributed as dist
        self.torch, self.dist = torch, dist
        self.n, self.k, self.p, self.rank = n, k, world, rank
        self.c = c or grid_c(world)
        if world % (self.c * self.c):
            raise ValueError(f"c={self.c} needs c^2 | p (p={world})")
        c = self.c
        self.q = world // c                  # grid rows (p/c)
        self.rounds = self.q // c            # p/c^2 rounds
        self.i, self.j = divmod(rank, c)
        self.B = tile_bounds(n, self.q)
        i, j, B = self.i, self.j, self.B
        # groups: every rank creates every group in the same order (torch.distributed requirement)
        self.col_group = self.row_group = None
        for jj in range(c):
            g = dist.new_group([ii * c + jj for ii in range(self.q)]) if self.q > 1 else None
            if jj == j:
                self.col_group = g
        for ii in range(self.q):
            g = dist.new_group([ii * c + jj for jj in range(c)]) if c > 1 else None
            if ii == i:
                self.row_group = g
        # my A pieces: row block i x X tile t, for the p/c^2 tiles t of column block j
        rp = np.asarray(row_ptr, dtype=np.int64)
        cl = np.asarray(col, dtype=np.int64)
        vl = np.asarray(val)
        r0, r1 = B[i], B[i + 1]
        lo, hi = rp[r0], rp[r1]
        rows = np.repeat(np.arange(r1 - r0, dtype=np.int64), np.diff(rp[r0:r1 + 1]))
        ccol, cval = cl[lo:hi], vl[lo:hi]
        self.tiles = []                      # (t, src rank, CSR piece)
        for r in range(self.rounds):
            t = j * self.rounds + r
            m = (ccol >= B[t]) & (ccol < B[t + 1])
            pr, pc, pv = rows[m], ccol[m] - B[t], cval[m]
            ptr = np.zeros(r1 - r0 + 1, dtype=np.int64)
            np.add.at(ptr, pr + 1, 1)
            A = torch.sparse_csr_tensor(torch.from_numpy(np.cumsum(ptr)).to(device), torch.from_numpy(pc).to(device),
                                        torch.from_numpy(np.ascontiguousarray(pv)).to(device=device, dtype=torch_dtype),
                                        size=(r1 - r0, B[t + 1] - B[t]))
            self.tiles.append((t, t * c + j, A))
        self.maxrows = max(B[t + 1] - B[t] for t in range(self.q))
        self.buf = torch.empty((self.maxrows, k), dtype=torch_dtype, device=device)
        self.Y = torch.empty((r1 - r0, k), dtype=torch_dtype, device=device)

    @property
    def row_range(self):
        return self.B[self.i], self.B[self.i + 1]

    def step(self, X_tile):
        """X_tile: this grid row's X tile (rows row_range); returns the Y tile (same rows)."""
        torch, dist = self.torch, self.dist
        self.Y.zero_()
        for t, src, A in self.tiles:
            rows_t = self.B[t + 1] - self.B[t]
            buf = self.buf[:rows_t]
            if src == self.rank:
                buf.copy_(X_tile)
            if self.col_group is not None:
                dist.broadcast(buf, src=src, group=self.col_group)
            self.Y.add_(torch.sparse.mm(A, buf))
        if self.row_group is not None:
            dist.all_reduce(self.Y, group=self.row_group)
        return self.Y

    def ledger(self, es: int) -> dict:
        return ledger(self.n, self.k, es, self.p, self.c, self.rank)
