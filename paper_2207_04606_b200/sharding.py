"""Row-partitioned multi-GPU SpMM plumbing.

Output rows are independent, so the hot path shards by contiguous, nnz-balanced row ranges
(`strata_partition_rows`: cut p is the first row whose indptr reaches nnz*p/P).  Each rank
decomposes and multiplies its shard on its own GPU with X replicated.  To overlap the only
collective (the NCCL all-gather that reassembles Y — the next GNN layer needs all of it) with
compute, every rank's range is further cut into `chunks` nnz-balanced sub-ranges: chunk c of
every rank lands in slot [c][rank] of a padded [chunks][P][max_rows][d] buffer, so chunk c's
all-gather can run while chunk c+1 is being computed.  `unpad` restores global row order.
"""
from __future__ import annotations

import numpy as np

from .ops import CsrMatrix, partition_rows


class RowShardPlan:
    def __init__(self, csr: CsrMatrix, world: int, chunks: int = 1):
        self.world = world
        self.chunks = chunks
        self.rows = csr.rows
        self.bounds = partition_rows(csr.indptr, world)
        self._csr = csr
        # sub[r][c] = (row0, row1) of chunk c of rank r, balanced by nnz inside the rank range
        self.sub = []
        for r in range(world):
            r0, r1 = int(self.bounds[r]), int(self.bounds[r + 1])
            local = partition_rows(csr.indptr[r0:r1 + 1] - csr.indptr[r0], chunks) + r0
            self.sub.append([(int(local[c]), int(local[c + 1])) for c in range(chunks)])
        self.max_rows = max((b - a for rr in self.sub for (a, b) in rr), default=0)
        self.max_rows = max(self.max_rows, 1)

    def rows_of(self, rank: int):
        return int(self.bounds[rank]), int(self.bounds[rank + 1])

    def shard(self, rank: int) -> CsrMatrix:
        r0, r1 = self.rows_of(rank)
        return self._csr.row_slice(r0, r1)

    def chunk(self, rank: int, c: int) -> CsrMatrix:
        a, b = self.sub[rank][c]
        return self._csr.row_slice(a, b)

    def chunk_rows(self, rank: int, c: int) -> int:
        a, b = self.sub[rank][c]
        return b - a

    def shard_nnz(self, rank: int) -> int:
        r0, r1 = self.rows_of(rank)
        return int(self._csr.indptr[r1] - self._csr.indptr[r0])

    @property
    def padded_rows(self) -> int:
        return self.chunks * self.world * self.max_rows

    def slot(self, c: int, rank: int) -> int:
        """First row of slot [c][rank] in the padded gathered buffer."""
        return (c * self.world + rank) * self.max_rows

    def unpad(self, y_padded):
        """[chunks*P*max_rows][d] gathered buffer -> [rows][d] in global row order."""
        parts = []
        for r in range(self.world):
            for c in range(self.chunks):
                s = self.slot(c, r)
                parts.append(y_padded[s: s + self.chunk_rows(r, c)])
        if isinstance(y_padded, np.ndarray):
            return np.concatenate(parts, axis=0)
        import torch
        return torch.cat(parts, dim=0)
