"""Pins for the shard oracle."""
import numpy as np
import pytest

from oracle import shard as S
from oracle import tree as T
from synth import workloads as W
from tests.helpers import random_workload


def _runs(sigma, req_shard, g):
    pos = [k for k, r in enumerate(sigma) if req_shard[r] == g]
    runs = 0
    for i, k in enumerate(pos):
        if i == 0 or pos[i - 1] != k - 1:
            runs += 1
    return runs, pos


@pytest.mark.parametrize("seed", range(8))
def test_g1_identity_and_fold(seed):
    w = random_workload(seed, n_req=12)
    v = T.build(w)
    assert np.all(S.shard_assign(w, v, 1) == 0)
    for G in (2, 3):
        rs = S.shard_assign(w, v, G)
        assert rs.shape == (w.n_req,) and set(rs.tolist()) <= set(range(G))
        sigma = list(v["dfs_order"])
        # shard g = block g U block 2G-1-g: at most two contiguous runs of sigma,
        # and shards appear in the fold order 0,1,..,G-1,G-1,..,1,0 along sigma
        seq = [int(rs[r]) for r in sigma]
        for g in range(G):
            assert _runs(sigma, rs, g)[0] <= 2
        collapsed = [x for i, x in enumerate(seq) if i == 0 or seq[i - 1] != x]
        fold = list(range(G)) + list(range(G - 1, -1, -1))
        it = iter(fold)
        assert all(any(x == y for y in it) for x in collapsed)     # subsequence of the fold


def test_weights_conserved_and_balanced():
    w = W.c2_mmlu_decode()
    v = T.build(w)
    sigma, wt = S.weights(w, v, 213)
    Wtot = sum(wt.values())
    for G in (2, 4, 8):
        rs = S.shard_assign(w, v, G)
        per = [sum(wt[r] for r in sigma if rs[r] == g) for g in range(G)]
        assert sum(per) == Wtot
        # the first-touch of the shared 1024-token node lands on one shard only
        assert max(per) / (Wtot / G) < 1.6


def test_first_touch_counts_shared_node_once():
    w = W.c2_mmlu_decode()
    v = T.build(w)
    sigma, wt = S.weights(w, v, 1)
    D, Hq, Hkv = 128, 32, 8
    flops = sum(4 * D * Hq * int(np.diff(w.tok_off)[r]) for r in range(w.n_req))
    kv = int(v["node_len"].sum()) * Hkv * D * 2 * 2
    assert sum(wt.values()) == flops + kv


def test_c5_two_documents_per_gpu():
    # subtree snapping yields 2 whole documents per GPU at G=8
    w = W.c5_70b_32k()
    v = T.build(w)
    rs = S.shard_assign(w, v, 8)
    doc = np.arange(w.n_req) // 64
    for g in range(8):
        docs = set(doc[rs == g].tolist())
        assert len(docs) == 2
        for dd in docs:
            assert np.all(rs[doc == dd] == g)        # whole documents


def test_shard_trees_restrict():
    w = random_workload(4, n_req=12)
    v = T.build(w)
    rs = S.shard_assign(w, v, 2)
    subs = S.shard_workloads(w, rs, 2)
    assert sum(s.n_req for s in subs) == w.n_req
    for s in subs:
        assert list(s.global_id) == sorted(s.global_id)
        T.build(s)


def test_cut_targets_round_up():
    # §8(c-3) step 3: tau_i = ceil(i W / 2G).  G = 1, W = 7: tau = 4, and the only prefix
    # sum within the window |S_k - tau| * 32 <= 7 is S_2 = 4 (a round-down target 3 would
    # have no candidate and tie S_1 = 2 / S_2 = 4, taking k = 1).
    assert S.cut_points([0, 2, 4, 7], [0, 0, 0, 0], 1) == [0, 2, 3]
    # G = 2, W = 10: tau = 3, 5, 8 (ceil of 2.5, 5, 7.5)
    assert S.cut_points([0, 3, 5, 7, 8, 10], [0] * 6, 2) == [0, 1, 2, 4, 5]


def test_cut_prefers_subtree_boundary_in_window():
    # step 4: inside the window the smallest lcp wins over the closest prefix sum
    Ssum = [0] + list(range(10, 330, 10))                  # W = 320, G = 1: tau = 160, window +-10
    lcp = [0] + [5] * 31 + [0]
    lcp[17] = 1                                          # S_17 = 170 is 10 from tau
    assert S.cut_points(Ssum, lcp, 1) == [0, 17, 32]
    lcp[15] = 1                                          # S_15 = 150, also 10 from tau
    assert S.cut_points(Ssum, lcp, 1) == [0, 15, 32]       # |150-160| = |170-160|: smaller k
    lcp[16] = 1
    assert S.cut_points(Ssum, lcp, 1) == [0, 16, 32]       # exact hit at equal lcp


def test_cuts_fallback_heavy_request():
    # step 4 fallback (no prefix sum in the window): nearest prefix sum, ties to the smaller
    # k.  One heavy request (weight 99 of W = 101) spans targets tau = 13, 26, 38, 51, 64,
    # 76, 89 (G = 4); |1 - 51| = 50 > |100 - 51| = 49 moves the cut past it at i = 4.
    assert S.cut_points([0, 1, 100, 101], [0, 0, 0, 0], 4) == [0, 1, 1, 1, 2, 2, 2, 2, 3]
