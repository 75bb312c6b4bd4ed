"""GPU: the fused SpMM + all-gather over peer memory (strata_spmm_hyb_f32_multi +
sharding.PeerAllGather).

* single process: the multi-destination store path (main kernel, split-run fix-up, empty rows,
  the c > 1 f64 accumulator) writes bit-identical rows to every destination;
* two processes on one GPU (the only GPU a test box has): each rank decomposes its nnz-balanced
  row shard, exchanges CUDA IPC handles of its full-size Y replica through a gloo group, and its
  SpMM stores every row into both replicas — each replica must equal the oracle bitwise.  Two
  processes exercise exactly the cross-process mapping one-process-per-GPU ranks use (IPC
  handle + offset, peer-mapped stores); on an 8-GPU node the stores travel over NVLink."""
import os
import socket

import numpy as np
import pytest
import torch

import paper_2207_04606_b200 as S
from oracle import port

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.mark.parametrize("c,d", [(1, 64), (1, 128), (3, 32), (1, 24)])
def test_spmm_multi_destinations_single_process(cuda, c, d):
    m = S.generate_matrix("powerlaw", 12000, 11000, 0, 0, 0, 14.0, 4)  # long + empty rows
    h = S.decompose_hyb(m.to_device(cuda), c, 3)  # k = 3 forces split rows
    X = torch.from_numpy(S.dense_int((m.cols, d), 8)).to(cuda)
    ref = S.spmm(h, X)
    outs = [torch.full((m.rows, d), float("nan"), device=cuda) for _ in range(3)]
    S.spmm_multi(h, X, [o.data_ptr() for o in outs])
    for o in outs:
        assert torch.equal(o, ref)
    want = port.spmm_csr_refnum(m.rows, m.indptr, m.indices, m.values, X.cpu().numpy())
    assert np.array_equal(ref.cpu().numpy(), want)
    with pytest.raises(S.StrataError):
        S.spmm_multi(h, X, [outs[0].data_ptr()] * 9)


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _peer_worker(rank, world, port, q):
    import sys
    sys.path.insert(0, ROOT)
    import torch
    import torch.distributed as dist
    import paper_2207_04606_b200 as S
    from paper_2207_04606_b200.sharding import PeerAllGather, RowShardPlan
    from oracle import port as P
    try:
        torch.cuda.set_device(0)
        dev = torch.device("cuda:0")
        dist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{port}", rank=rank,
                                world_size=world)
        m = S.generate_matrix("powerlaw", 20000, 18000, 0, 0, 0, 12.0, 6)
        d = 64
        plan = RowShardPlan(m, world)
        r0, r1 = plan.rows_of(rank)
        h = S.decompose_hyb(plan.shard(rank).to_device(dev), 1, S.hyb_auto_k(m))
        X = torch.from_numpy(S.dense_int((m.cols, d), 9)).to(dev)
        y_full = torch.full((m.rows, d), float("nan"), device=dev)
        pag = PeerAllGather(y_full, rank, world)
        torch.cuda.synchronize()
        dist.barrier()
        S.spmm_multi(h, X, pag.dsts(r0))
        torch.cuda.synchronize()
        dist.barrier()  # every rank's stores are complete
        want = P.spmm_csr_refnum(m.rows, m.indptr, m.indices, m.values, X.cpu().numpy())
        ok = bool(np.array_equal(y_full.cpu().numpy(), want))
        dist.barrier()  # peers stop touching this replica before it is unmapped / freed
        pag.close()
        dist.destroy_process_group()
        q.put((rank, ok, ""))
    except Exception as e:  # surface the failure in the parent
        q.put((rank, False, repr(e)))


def test_peer_allgather_two_processes_one_gpu(cuda):
    import torch.multiprocessing as mp
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port_ = _free_port()
    procs = [ctx.Process(target=_peer_worker, args=(r, 2, port_, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = [q.get(timeout=300) for _ in procs]
    for p in procs:
        p.join(timeout=60)
    assert all(ok for _, ok, _ in res), res
