"""CPU suite: executable model of the hyb SpMM schedule (paper_2207_04606_b200/csrc/spmm_hyb.cu
+ the run planner in hyb_build.cu).

The device kernel splits every ELL part into chunks of 256 slots (whole rows), produces each
output row in exactly one virtual warp, and routes the partial sums of split rows whose
segments cross chunk boundaries through a carry buffer that a fixed-order fix-up reduces.
This model replays that exact plan (chunk size, head/tail carry rule, run detection with the
"uniform chunk" condition, tile/level-2 fix-up order) in float64 on the oracle's
decomposition and must reproduce the reference output bit for bit on integer data."""
import numpy as np
import pytest

from oracle import port

FIX_TILE = 32  # kFixTile in capi_internal.h


def model_spmm(rows, parts, X, k):
    d = X.shape[1]
    Y = np.zeros((rows, d))
    for P in parts:
        b = P["bucket"]
        W = 1 << b
        rpc = 1 << max(0, 8 - b)
        nr, I, J, V = P["nrows"], P["I_indices"], P["J_indices"], P["values"]
        nch = (nr + rpc - 1) // rpc
        split = b == k
        carry = np.zeros((nch, 2, d))
        for ch in range(nch):
            r0, r1 = ch * rpc, min(ch * rpc + rpc, nr)
            head = split and ch > 0 and I[r0 - 1] == I[r0]
            tail = split and ch + 1 < nch and I[r1 - 1] == I[r1]
            acc, cur, first = np.zeros(d), None, True

            def flush(final):
                if split and first and head:
                    carry[ch, 0] = acc
                elif split and final and tail:
                    carry[ch, 1] = acc
                else:
                    Y[cur] = acc

            for r in range(r0, r1):
                if cur is not None and I[r] != cur:
                    flush(False)
                    first, acc = False, np.zeros(d)
                cur = I[r]
                for s in range(W):
                    t = r * W + s
                    if s > 0 and J[t] == J[t - 1]:
                        continue  # pad slot (storage.cpp:528 rule)
                    acc = acc + V[t] * X[J[t]]
            flush(True)
        if not split or nch < 2:
            continue

        def cross(cc):
            return 0 <= cc < nch - 1 and I[(cc + 1) * rpc - 1] == I[(cc + 1) * rpc]

        def uniform(cc):
            return I[cc * rpc] == I[min((cc + 1) * rpc, nr) - 1]

        starts = [c for c in range(nch) if cross(c) and not (cross(c - 1) and uniform(c))]
        ends = [c for c in range(nch) if cross(c - 1) and not (cross(c) and uniform(c))]
        assert len(starts) == len(ends)
        for ca, cb in zip(starts, ends):
            row = I[(ca + 1) * rpc - 1]
            contrib = [carry[ca, 1]] + [carry[c, 0] for c in range(ca + 1, cb + 1)]
            tiles = [sum(contrib[u:u + FIX_TILE], np.zeros(d)) for u in range(0, len(contrib), FIX_TILE)]
            Y[row] = sum(tiles, np.zeros(d))
    return Y.astype(np.float32)


@pytest.mark.parametrize("seed", range(12))
def test_schedule_model_matches_reference(seed):
    rng = np.random.default_rng(seed)
    import paper_2207_04606_b200 as S
    n = int(rng.integers(200, 3000))
    m = S.generate_matrix("powerlaw", n, int(rng.integers(100, 3000)), 0, 0, 0,
                          float(rng.uniform(2, 60)), seed + 1)
    k = int(rng.integers(0, 6))
    parts, _ = port.hyb_decompose(m.rows, m.cols, m.indptr, m.indices, m.values, 1, k)
    X = S.dense_int((m.cols, 4), seed)
    want = port.spmm_csr_refnum(m.rows, m.indptr, m.indices, m.values, X)
    assert np.array_equal(model_spmm(m.rows, parts, X.astype(np.float64), k), want)
