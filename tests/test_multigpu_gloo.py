"""CPU suite: the N > 1 path's host logic on a world-size-2 `gloo` group.

Each rank takes its nnz-balanced row shard (RowShardPlan, the code bench.py runs under
torchrun), decomposes and multiplies it (here with the oracle, since there is no GPU), places
its rows in slot `rank` of the padded buffer, and the all-gather + unpad must reassemble the
global result bit for bit.  Also checks SURVEY §7's property that per-shard hyb decompositions
concatenated per bucket, in shard order, equal the global decomposition."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, out_path):
    import sys
    sys.path.insert(0, ROOT)
    import paper_2207_04606_b200 as S
    from paper_2207_04606_b200.sharding import RowShardPlan
    from oracle import port as P

    dist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{port}", rank=rank,
                            world_size=world)
    m = S.generate_matrix("powerlaw", 6000, 5000, 0, 0, 0, 20.0, 3)
    plan = RowShardPlan(m, world, chunks=3)  # bench.py's overlapped layout
    k = S.hyb_auto_k(m)
    X = S.dense_int((m.cols, 16), 5)
    full_buf = torch.zeros((plan.padded_rows, 16), dtype=torch.float32)
    for c in range(plan.chunks):  # chunk c computed, then its all-gather (async on a GPU)
        sh = plan.chunk(rank, c)
        parts, _ = P.hyb_decompose(sh.rows, sh.cols, sh.indptr, sh.indices, sh.values, 1, k)
        y = P.spmm_hyb_refnum(sh.rows, parts, X)
        buf = torch.zeros((plan.max_rows, 16), dtype=torch.float32)
        buf[: sh.rows] = torch.from_numpy(y)
        gathered = [torch.empty_like(buf) for _ in range(world)]
        dist.all_gather(gathered, buf)
        s0 = plan.slot(c, 0)
        full_buf[s0: s0 + world * plan.max_rows] = torch.cat(gathered, 0)
    full = plan.unpad(full_buf).numpy()
    if rank == 0:
        np.save(out_path, full)
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("world", [2])
def test_row_sharded_spmm_allgather_gloo(tmp_path, world):
    import paper_2207_04606_b200 as S
    from oracle import port as P
    out = str(tmp_path / "y.npy")
    mp.spawn(_worker, args=(world, _free_port(), out), nprocs=world, join=True)
    m = S.generate_matrix("powerlaw", 6000, 5000, 0, 0, 0, 20.0, 3)
    X = S.dense_int((m.cols, 16), 5)
    want = P.spmm_csr_refnum(m.rows, m.indptr, m.indices, m.values, X)
    assert np.array_equal(np.load(out), want)


def _bcast_worker(rank, world, port, out_path):
    """The native sharded plan's reassembly (shard.cu): per chunk, every rank's rows are
    broadcast from their owner into the full in-place Y (grouped ncclBroadcast on the GPU,
    dist.broadcast over gloo here); the SDDMM's contiguous nnz ranges likewise into B."""
    import sys
    sys.path.insert(0, ROOT)
    import paper_2207_04606_b200 as S
    from paper_2207_04606_b200.sharding import RowShardPlan
    from oracle import port as P

    dist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{port}", rank=rank,
                            world_size=world)
    m = S.generate_matrix("powerlaw", 7000, 6500, 0, 0, 0, 18.0, 4)
    plan = RowShardPlan(m, world, chunks=3)  # the same cuts strata_shard_plan_create makes
    d = 8
    X = S.dense_int((m.cols, d), 6)
    Y = torch.full((m.rows, d), float("nan"))
    for c in range(plan.chunks):
        a, b = plan.sub[rank][c]
        sh = plan.chunk(rank, c)
        Y[a:b] = torch.from_numpy(P.spmm_csr_refnum(sh.rows, sh.indptr, sh.indices, sh.values, X))
        for q in range(world):  # one group: chunk c of every rank, from its owner, in place
            qa, qb = plan.sub[q][c]
            seg = Y[qa:qb].contiguous()
            dist.broadcast(seg, src=q)
            Y[qa:qb] = seg
    Xs = S.dense_int((m.rows, d), 7)
    Yd = S.dense_int((d, m.cols), 8)
    B = torch.full((m.nnz,), float("nan"))
    r0, r1 = plan.rows_of(rank)
    q0, q1 = int(m.indptr[r0]), int(m.indptr[r1])
    sh = plan.shard(rank)
    B[q0:q1] = torch.from_numpy(P.sddmm_csr_refnum(sh.rows, sh.cols, sh.indptr, sh.indices,
                                                   sh.values, Xs[r0:r1], Yd))
    for q in range(world):
        qr0, qr1 = plan.rows_of(q)
        a, b = int(m.indptr[qr0]), int(m.indptr[qr1])
        seg = B[a:b].contiguous()
        dist.broadcast(seg, src=q)
        B[a:b] = seg
    np.save(out_path + f".{rank}.y.npy", Y.numpy())
    np.save(out_path + f".{rank}.b.npy", B.numpy())
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3])
def test_sharded_broadcast_reassembly_gloo(tmp_path, world):
    import paper_2207_04606_b200 as S
    from oracle import port as P
    out = str(tmp_path / "r")
    mp.spawn(_bcast_worker, args=(world, _free_port(), out), nprocs=world, join=True)
    m = S.generate_matrix("powerlaw", 7000, 6500, 0, 0, 0, 18.0, 4)
    wantY = P.spmm_csr_refnum(m.rows, m.indptr, m.indices, m.values, S.dense_int((m.cols, 8), 6))
    wantB = P.sddmm_csr_refnum(m.rows, m.cols, m.indptr, m.indices, m.values,
                               S.dense_int((m.rows, 8), 7), S.dense_int((8, m.cols), 8))
    for r in range(world):
        assert np.array_equal(np.load(out + f".{r}.y.npy"), wantY)
        assert np.array_equal(np.load(out + f".{r}.b.npy"), wantB)


def _id_worker(rank, world, port, out_path):
    import sys
    sys.path.insert(0, ROOT)
    from paper_2207_04606_b200.sharding import NcclComm
    dist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{port}", rank=rank,
                            world_size=world)
    uid = NcclComm.exchange_unique_id(rank, world, make_id=lambda: bytes(range(128)))
    with open(out_path + f".{rank}", "wb") as f:
        f.write(uid)
    dist.barrier()
    dist.destroy_process_group()


def test_nccl_unique_id_exchange_gloo(tmp_path):
    """The NCCL bootstrap of the native sharded path: rank 0's ncclUniqueId reaches every rank."""
    out = str(tmp_path / "id")
    mp.spawn(_id_worker, args=(3, _free_port(), out), nprocs=3, join=True)
    for r in range(3):
        assert open(out + f".{r}", "rb").read() == bytes(range(128))


@pytest.mark.parametrize("parts", [2, 3, 5, 8])
def test_shard_decompositions_concatenate_to_global(parts):
    import paper_2207_04606_b200 as S
    from paper_2207_04606_b200.sharding import RowShardPlan
    from oracle import port as P
    m = S.generate_matrix("powerlaw", 8000, 8000, 0, 0, 0, 30.0, 1)
    k = S.hyb_auto_k(m)
    for c in (1, 3):
        glob, _ = P.hyb_decompose(m.rows, m.cols, m.indptr, m.indices, m.values, c, k)
        plan = RowShardPlan(m, parts)
        cat = {}
        for r in range(parts):
            sh = plan.shard(r)
            r0, _ = plan.rows_of(r)
            sp, _ = P.hyb_decompose(sh.rows, sh.cols, sh.indptr, sh.indices, sh.values, c, k)
            for p in sp:
                key = (p["partition"], p["bucket"])
                e = cat.setdefault(key, {"I": [], "J": [], "V": []})
                e["I"].append(p["I_indices"] + r0)
                e["J"].append(p["J_indices"])
                e["V"].append(p["values"])
        assert sorted(cat) == [(p["partition"], p["bucket"]) for p in glob]
        for p in glob:
            e = cat[(p["partition"], p["bucket"])]
            assert np.array_equal(np.concatenate(e["I"]), p["I_indices"])
            assert np.array_equal(np.concatenate(e["J"]), p["J_indices"])
            assert np.array_equal(np.concatenate(e["V"]), p["values"])


def test_partition_covers_rows_and_balances():
    import paper_2207_04606_b200 as S
    from paper_2207_04606_b200.sharding import RowShardPlan
    m = S.generate_matrix("powerlaw", 50000, 50000, 0, 0, 0, 25.3, 1)
    for world in (1, 2, 4, 8):
        plan = RowShardPlan(m, world)
        assert sum(plan.shard(r).rows for r in range(world)) == m.rows
        nnz = [plan.shard_nnz(r) for r in range(world)]
        assert sum(nnz) == m.nnz
        assert max(nnz) <= m.nnz / world + np.diff(m.indptr).max()
