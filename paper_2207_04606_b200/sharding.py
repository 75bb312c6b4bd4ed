"""Row-partitioned multi-GPU SpMM plumbing.

Output rows are independent, so the hot path shards by contiguous, nnz-balanced row ranges
(`strata_partition_rows`: cut p is the first row whose indptr reaches nnz*p/P).  Each rank
decomposes and multiplies its shard on its own GPU with X replicated, writes its rows into slot
`rank` of a padded [P * max_rows][d] buffer, and one NCCL all-gather (the only collective: the
next GNN layer needs all of Y) reassembles Y on every rank; `unpad` drops the padding rows.
"""
from __future__ import annotations

import numpy as np

from .ops import CsrMatrix, partition_rows


class RowShardPlan:
    def __init__(self, csr: CsrMatrix, world: int):
        self.world = world
        self.rows = csr.rows
        self.bounds = partition_rows(csr.indptr, world)
        self.max_rows = int(np.max(np.diff(self.bounds))) if world > 0 else 0
        self._csr = csr

    def rows_of(self, rank: int):
        return int(self.bounds[rank]), int(self.bounds[rank + 1])

    def shard(self, rank: int) -> CsrMatrix:
        r0, r1 = self.rows_of(rank)
        return self._csr.row_slice(r0, r1)

    def shard_nnz(self, rank: int) -> int:
        r0, r1 = self.rows_of(rank)
        return int(self._csr.indptr[r1] - self._csr.indptr[r0])

    @property
    def padded_rows(self) -> int:
        return self.max_rows * self.world

    def unpad(self, y_padded):
        """[P*max_rows][d] gathered buffer -> [rows][d] (rank slots concatenated in order)."""
        parts = []
        for r in range(self.world):
            r0, r1 = self.rows_of(r)
            parts.append(y_padded[r * self.max_rows: r * self.max_rows + (r1 - r0)])
        if isinstance(y_padded, np.ndarray):
            return np.concatenate(parts, axis=0)
        import torch
        return torch.cat(parts, dim=0)
