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

import ctypes as C

from ._lib import check, lib
from .ops import CsrMatrix, DeviceCsr, _dense, _ptr, _stream, partition_rows


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


class PeerAllGather:
    """Fused SpMM + all-gather over peer memory (one process per GPU).

    Every rank owns a full [rows][d] f32 replica of Y.  The replicas' CUDA IPC handles are
    exchanged once through the process group; each rank then runs its shard's SpMM with
    ``ops.spmm_multi`` storing every finished row into all replicas (its own plus the peers',
    written over NVLink), so the reassembly traffic leaves the SMs as rows are produced — no
    separate collective, no padded buffer, global row order directly.  ``fence()`` (a
    one-element all-reduce on the stream) orders the next layer's reads after every rank's
    stores.
    """

    def __init__(self, y_full, rank: int, world: int, group=None):
        import torch.distributed as dist
        from .ops import ipc_handle, ipc_open
        import torch
        self.y = y_full
        self.rank, self.world, self.group = rank, world, group
        self.d = int(y_full.shape[1])
        self.ptrs, self._opened = [], []

        def agree(ok: bool, what: str, err):
            # every rank takes the same branch: a failure on any rank raises on all of them,
            # so callers that fall back to NCCL keep their collectives in step
            t = torch.tensor([1 if ok else 0], dtype=torch.int32, device=y_full.device)
            dist.all_reduce(t, op=dist.ReduceOp.MIN, group=group)
            if int(t[0]) != 1:
                self.close()
                raise RuntimeError(f"{what} failed on a rank" + (f": {err}" if err else ""))

        mine, err = None, None
        try:
            mine = ipc_handle(y_full)
        except Exception as e:  # noqa: BLE001
            err = e
        agree(mine is not None, "CUDA IPC handle export", err)
        handles = [None] * world
        dist.all_gather_object(handles, mine, group=group)
        err = None
        try:
            for r, (hd, off) in enumerate(handles):
                if r == rank:
                    self.ptrs.append(y_full.data_ptr())
                else:
                    base = ipc_open(hd)
                    self._opened.append(base)
                    self.ptrs.append(base + off)
        except Exception as e:  # noqa: BLE001
            err = e
        agree(err is None, "CUDA IPC peer mapping", err)
        self._flag = torch.zeros(1, dtype=torch.int32, device=y_full.device)

    def dsts(self, row0: int):
        """Destination addresses of global row ``row0`` in every replica."""
        return [p + row0 * self.d * 4 for p in self.ptrs]

    def fence(self):
        import torch.distributed as dist
        dist.all_reduce(self._flag, group=self.group)

    def close(self):
        from .ops import ipc_close
        for p in self._opened:
            ipc_close(p)
        self._opened = []


class NcclComm:
    """An NCCL communicator created through the C ABI (strata_nccl_comm_init): rank 0 draws
    the unique id, the process group broadcasts it, every rank joins.  ``ptr`` is the address
    of the ncclComm_t the sharded entry points take."""

    @staticmethod
    def exchange_unique_id(rank: int, world: int, group=None, make_id=None) -> bytes:
        """Rank 0's ncclUniqueId (128 bytes) on every rank (an object broadcast: works on gloo
        and NCCL process groups alike)."""
        import torch.distributed as dist
        uid = b""
        if rank == 0:
            if make_id is not None:
                uid = make_id()
            else:
                idb = (C.c_char * 128)()
                check(lib.strata_nccl_unique_id(idb))
                uid = bytes(idb.raw)
        if world > 1:
            box = [uid]
            dist.broadcast_object_list(box, src=0, group=group)
            uid = box[0]
        return uid

    def __init__(self, rank: int, world: int, group=None):
        idb = (C.c_char * 128).from_buffer_copy(self.exchange_unique_id(rank, world, group))
        self._comm = C.c_void_p()
        check(lib.strata_nccl_comm_init(idb, world, rank, C.byref(self._comm)))
        self.rank, self.world = rank, world

    @property
    def ptr(self) -> int:
        return C.addressof(self._comm)

    def close(self):
        if self._comm:
            lib.strata_nccl_comm_destroy(C.byref(self._comm))
            self._comm = C.c_void_p()


class ShardPlan:
    """Native row-partitioned plan (strata_shard_plan_create): this rank's nnz-balanced row
    range, cut into ``chunks`` sub-ranges, each decomposed to hyb(c, k) on the device.  The
    DeviceCsr must outlive the plan (the sharded SDDMM reads its arrays)."""

    def __init__(self, csr: DeviceCsr, rank: int, world: int, chunks: int = 1, c: int = 1,
                 k: int = None, stream=None):
        from .ops import hyb_auto_k
        self.csr = csr
        self.rank, self.world, self.chunks = rank, world, chunks
        self.rows, self.cols, self.nnz = csr.rows, csr.cols, csr.nnz
        k = hyb_auto_k(csr) if k is None else k
        self._h = C.c_void_p()
        check(lib.strata_shard_plan_create(_ptr(csr.indptr), _ptr(csr.indices), _ptr(csr.values),
                                           csr.rows, csr.cols, rank, world, chunks, c, k,
                                           C.byref(self._h), _stream(stream)))

    def rows_of(self, rank: int, chunk: int = -1):
        a, b = C.c_int64(), C.c_int64()
        check(lib.strata_shard_plan_rows(self._h, rank, chunk, C.byref(a), C.byref(b)))
        return a.value, b.value

    def spmm(self, X, Y, comm: "NcclComm" = None, stream=None):
        """Y[rows][d] replica on every rank; comm=None only at world 1."""
        d = int(X.shape[1])
        _dense(X, "X", (self.cols, d), "f32", X.device)
        _dense(Y, "Y", (self.rows, d), "f32", X.device)
        check(lib.strata_spmm_hyb_f32_sharded(self._h, _ptr(X), _ptr(Y), d,
                                              comm.ptr if comm else None, self.world,
                                              _stream(stream)))
        return Y

    def spmm_p2p(self, X, dst_ptrs, d: int, stream=None):
        """Fused peer stores: dst_ptrs[q] = base address of rank q's Y replica."""
        _dense(X, "X", (self.cols, d), "f32", X.device)
        arr = (C.c_void_p * len(dst_ptrs))(*dst_ptrs)
        check(lib.strata_spmm_hyb_f32_sharded_p2p(self._h, _ptr(X), arr, len(dst_ptrs), d,
                                                  _stream(stream)))

    def sddmm(self, X, Yd, B, gather: bool = True, comm: "NcclComm" = None, stream=None):
        d = int(X.shape[1])
        _dense(X, "X", (self.rows, d), "f32", X.device)
        _dense(Yd, "Y", (d, self.cols), "f32", X.device)
        _dense(B, "B", (self.nnz,), "f32", X.device)
        check(lib.strata_sddmm_csr_f32_sharded(self._h, _ptr(X), _ptr(Yd), _ptr(B), d,
                                               1 if gather else 0, comm.ptr if comm else None,
                                               self.world, _stream(stream)))
        return B

    def close(self):
        if self._h:
            lib.strata_shard_plan_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass
