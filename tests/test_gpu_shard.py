"""GPU: the native row-partitioned SpMM / SDDMM (strata_shard_plan_*, strata_*_sharded; SURVEY
§8b, §8e).

* world 1 through a real one-rank NCCL communicator made by the C ABI (and with comm = NULL):
  chunked plans (the per-chunk grouped broadcasts run on the plan's stream) must reproduce the
  single-GPU SpMM / SDDMM bit for bit;
* two processes on one GPU (the only GPU a test box has; NCCL refuses two ranks on one device):
  world-2 plans, the fused peer-store SpMM into both ranks' replicas through CUDA IPC, and the
  sharded SDDMM ranges (gather = 0) — every replica / range equal to the oracle bitwise;
* the plan's cuts equal strata_partition_rows' rule (the Python RowShardPlan's)."""
import os
import socket

import numpy as np
import pytest
import torch

import paper_2207_04606_b200 as S
from paper_2207_04606_b200.sharding import NcclComm, RowShardPlan, ShardPlan
from oracle import port

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.fixture(scope="module")
def comm1(cuda):
    c = NcclComm(0, 1)
    yield c
    c.close()


@pytest.mark.parametrize("chunks", [1, 3])
@pytest.mark.parametrize("use_comm", [True, False])
def test_sharded_spmm_sddmm_world1(cuda, comm1, chunks, use_comm):
    m = S.generate_matrix("powerlaw", 15000, 14000, 0, 0, 0, 13.0, 7)
    dm = m.to_device(cuda)
    plan = ShardPlan(dm, 0, 1, chunks=chunks)
    assert plan.rows_of(0) == (0, m.rows)
    # chunk cuts follow strata_partition_rows' rule inside the rank's range
    want_cuts = RowShardPlan(m, 1, chunks).sub[0]
    assert [plan.rows_of(0, c) for c in range(chunks)] == want_cuts
    comm = comm1 if use_comm else None
    d = 64
    X = torch.from_numpy(S.dense_int((m.cols, d), 3)).to(cuda)
    Y = torch.full((m.rows, d), float("nan"), device=cuda)
    plan.spmm(X, Y, comm)
    ref = S.spmm(S.decompose_hyb(dm, 1, S.hyb_auto_k(m)), X)
    assert torch.equal(Y, ref)
    assert np.array_equal(Y.cpu().numpy(),
                          port.spmm_csr_refnum(m.rows, m.indptr, m.indices, m.values, X.cpu().numpy()))
    Xs = torch.from_numpy(S.dense_int((m.rows, 32), 4)).to(cuda)
    Yd = torch.from_numpy(S.dense_int((32, m.cols), 5)).to(cuda)
    B = torch.full((m.nnz,), float("nan"), device=cuda)
    plan.sddmm(Xs, Yd, B, gather=True, comm=comm)
    assert torch.equal(B, S.sddmm(dm, Xs, Yd))


@pytest.mark.parametrize("c,k", [(2, 3), (3, 1)])
def test_sharded_column_partitions(cuda, comm1, c, k):
    """Chunks decomposed with c > 1 column partitions (f64 partition accumulation per chunk)
    and small k (split rows): the sharded SpMM equals the single-GPU hyb(c, k) SpMM bitwise."""
    m = S.generate_matrix("powerlaw", 9000, 8000, 0, 0, 0, 15.0, 2)
    dm = m.to_device(cuda)
    plan = ShardPlan(dm, 0, 1, chunks=3, c=c, k=k)
    X = torch.from_numpy(S.dense_int((m.cols, 64), 7)).to(cuda)
    Y = torch.full((m.rows, 64), float("nan"), device=cuda)
    plan.spmm(X, Y, comm1)
    assert torch.equal(Y, S.spmm(S.decompose_hyb(dm, c, k), X))


def test_sharded_errors(cuda, comm1):
    m = S.generate_matrix("powerlaw", 3000, 3000, 0, 0, 0, 6.0, 2)
    dm = m.to_device(cuda)
    p2 = ShardPlan(dm, 1, 2, chunks=2)
    X = torch.zeros((m.cols, 32), device=cuda)
    Y = torch.zeros((m.rows, 32), device=cuda)
    from paper_2207_04606_b200._lib import check, lib
    with pytest.raises(S.StrataError) as e:  # a one-rank communicator for a world-2 plan
        check(lib.strata_spmm_hyb_f32_sharded(p2._h, X.data_ptr(), Y.data_ptr(), 32, comm1.ptr, 2, 0))
    assert e.value.kind == "Usage" and "communicator is rank 0 of 1" in str(e.value)
    # comm = None: no reassembly, only this rank's rows are written
    Y.fill_(float("nan"))
    p2.spmm(X, Y, None)
    r0, r1 = p2.rows_of(1)
    assert not torch.isnan(Y[r0:r1]).any() and torch.isnan(Y[:r0]).all()
    with pytest.raises(S.StrataError) as e:
        check(lib.strata_spmm_hyb_f32_sharded(p2._h, X.data_ptr(), Y.data_ptr(), 32, None, 1, 0))
    assert "ndev 1 != plan world 2" in str(e.value)
    with pytest.raises(S.StrataError):
        ShardPlan(dm, 2, 2)


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port_, q):
    import sys
    sys.path.insert(0, ROOT)
    import torch
    import torch.distributed as dist
    import paper_2207_04606_b200 as S
    from paper_2207_04606_b200.sharding import PeerAllGather, ShardPlan
    from oracle import port as P
    try:
        torch.cuda.set_device(0)
        dev = torch.device("cuda:0")
        dist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{port_}", rank=rank,
                                world_size=world)
        m = S.generate_matrix("powerlaw", 20000, 18000, 0, 0, 0, 12.0, 6)
        dm = m.to_device(dev)
        plan = ShardPlan(dm, rank, world, chunks=2, k=3)
        d = 64
        X = torch.from_numpy(S.dense_int((m.cols, d), 9)).to(dev)
        y_full = torch.full((m.rows, d), float("nan"), device=dev)
        pag = PeerAllGather(y_full, rank, world)
        torch.cuda.synchronize()
        dist.barrier()
        plan.spmm_p2p(X, pag.dsts(0), d)
        torch.cuda.synchronize()
        dist.barrier()
        want = P.spmm_csr_refnum(m.rows, m.indptr, m.indices, m.values, X.cpu().numpy())
        ok_spmm = bool(np.array_equal(y_full.cpu().numpy(), want))
        # sharded SDDMM, B kept sharded: this rank's nnz range
        Xs = torch.from_numpy(S.dense_int((m.rows, 32), 4)).to(dev)
        Yd = torch.from_numpy(S.dense_int((32, m.cols), 5)).to(dev)
        B = torch.full((m.nnz,), float("nan"), device=dev)
        plan.sddmm(Xs, Yd, B, gather=False)
        r0, r1 = plan.rows_of(rank)
        q0, q1 = int(m.indptr[r0]), int(m.indptr[r1])
        wantB = P.sddmm_csr_refnum(m.rows, m.cols, m.indptr, m.indices, m.values,
                                   Xs.cpu().numpy(), Yd.cpu().numpy())
        Bh = B.cpu().numpy()
        ok_sddmm = bool(np.array_equal(Bh[q0:q1], wantB[q0:q1]) and np.isnan(Bh[:q0]).all()
                        and np.isnan(Bh[q1:]).all())
        # the two ranks' ranges tile [0, nnz)
        got = [None, None]
        dist.all_gather_object(got, (q0, q1))
        ok_tile = got[0][0] == 0 and got[0][1] == got[1][0] and got[1][1] == m.nnz
        dist.barrier()
        pag.close()
        dist.destroy_process_group()
        q.put((rank, ok_spmm and ok_sddmm and ok_tile, (ok_spmm, ok_sddmm, ok_tile)))
    except Exception as e:  # surface the failure in the parent
        q.put((rank, False, repr(e)))


def test_sharded_two_processes_one_gpu(cuda):
    import torch.multiprocessing as mp
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port_ = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port_, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = [q.get(timeout=300) for _ in procs]
    for p in procs:
        p.join(timeout=60)
    assert all(ok for _, ok, _ in res), res
