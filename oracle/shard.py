"""Shard oracle — independent re-implementation of `blend_shard`.

TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).

Follows PAPER P:246 (Data parallelism): "split continuous requests from both
sides of the prefix tree to different DP nodes.  Each block of requests has the
same amount of resource usage and maintains the same compute density as the
root node.  Since only the prompts along the split paths are recalculated, the
waste of prefix sharing is linear to the number of DP nodes."  Reading #20:

 1. sigma = request DFS order of the sorted tree.
 2. w_r = 4 D Hq sum_t (pos_t + 1) + kappa * first_touch_bytes(r), where
    first_touch counts each node's len*Hkv*D*2*b once, at its first request in sigma.
 3. S_k = prefix sums (S_0 = 0), W = S_R, targets tau_i = ceil(i W / 2G), i = 1..2G-1.
 4. cut k_i: among k in [0, R] with |S_k - tau_i| * 32G <= W minimise
    (lcp_tokens(sigma_{k-1}, sigma_k), |S_k - tau_i|, k)  [lcp = 0 at k = 0, R];
    no candidate -> argmin |S_k - tau_i| (ties -> smaller k); then k_i = max(k_i, k_{i-1}).
 5. blocks B_j = sigma[k_j : k_{j+1}]; shard g = B_g U B_{2G-1-g}.
 6. per-shard tree = the tree of the shard's requests in ascending global id order.
"""
from __future__ import annotations

import numpy as np

from . import tree as T


def _lcp(a: np.ndarray, b: np.ndarray) -> int:
    L = min(len(a), len(b))
    neq = np.nonzero(a[:L] != b[:L])[0]
    return int(neq[0]) if neq.size else L


def weights(w, view, kappa: int):
    R = w.n_req
    D, Hq, Hkv = w.head_dim, w.num_q_heads, w.num_kv_heads
    b = 2 if w.kv_dtype == "bf16" else 4
    sigma = [int(x) for x in view["dfs_order"]]
    n = np.diff(w.tok_off)
    touched = set()
    wt = {}
    for r in sigma:
        q = int(w.q_len[r])
        nr = int(n[r])
        flops = 4 * D * Hq * sum(nr - q + t + 1 for t in range(q))
        ft = 0
        for k in range(int(view["req_path_off"][r]), int(view["req_path_off"][r + 1])):
            node = int(view["req_path_nodes"][k])
            if node not in touched:
                touched.add(node)
                ft += int(view["node_len"][node]) * Hkv * D * 2 * b
        wt[r] = flops + kappa * ft
    return sigma, wt


def cut_points(S, lcp, G):
    """Steps 3-4: block boundaries k_0 = 0 <= k_1 <= ... <= k_{2G-1} <= k_{2G} = R over
    the prefix sums S[0..R] (S[0] = 0) and the lcp[k] of the pair (sigma_{k-1}, sigma_k)."""
    R = len(S) - 1
    W = S[-1]
    cuts = [0]
    for i in range(1, 2 * G):
        tau = -(-(i * W) // (2 * G))
        cands = [k for k in range(R + 1) if abs(S[k] - tau) * 32 * G <= W]
        if cands:
            k = min(cands, key=lambda k: (lcp[k], abs(S[k] - tau), k))
        else:
            k = min(range(R + 1), key=lambda k: (abs(S[k] - tau), k))
        cuts.append(max(k, cuts[-1]))
    cuts.append(R)
    return cuts


def shard_assign(w, view, n_shards: int, kappa: int = 213):
    """req_shard[R] (int32) for G = n_shards."""
    G = n_shards
    if G < 1:
        raise T.BlendError(T.EINVAL, "n_shards must be >= 1")
    sigma, wt = weights(w, view, kappa)
    R = len(sigma)
    S = [0]
    for r in sigma:
        S.append(S[-1] + wt[r])
    lcp = [0] * (R + 1)
    for k in range(1, R):
        lcp[k] = _lcp(w.path(sigma[k - 1]), w.path(sigma[k]))
    cuts = cut_points(S, lcp, G)
    req_shard = np.zeros(w.n_req, dtype=np.int32)
    for j in range(2 * G):
        g = j if j < G else 2 * G - 1 - j
        for r in sigma[cuts[j]:cuts[j + 1]]:
            req_shard[r] = g
    return req_shard


def shard_workloads(w, req_shard, n_shards, shard_free_pages=None):
    """Per-shard sub-workloads (requests in ascending global id order)."""
    from synth.workloads import Workload  # input container only
    out = []
    gid_all = w.global_id if w.global_id is not None else np.arange(w.n_req)
    for g in range(n_shards):
        rs = np.nonzero(req_shard == g)[0]
        paths = [w.path(int(r)) for r in rs]
        tok_off = np.zeros(len(rs) + 1, dtype=np.int64)
        tok_off[1:] = np.cumsum([len(x) for x in paths]) if len(rs) else []
        out.append(Workload(
            name=f"{w.name}_shard{g}", seed=w.seed, num_q_heads=w.num_q_heads,
            num_kv_heads=w.num_kv_heads, head_dim=w.head_dim, kv_dtype=w.kv_dtype,
            page_size=w.page_size, model_params=w.model_params, hidden=w.hidden, layers=w.layers,
            tokens=np.concatenate(paths).astype(np.int32) if paths else np.zeros(0, np.int32),
            tok_off=tok_off, q_len=w.q_len[rs], prompt_len=w.prompt_len[rs], out_len=w.out_len[rs],
            scale_q=w.scale_q,
            free_pages=None if shard_free_pages is None else shard_free_pages[g],
            global_id=np.asarray(gid_all)[rs].astype(np.int64)))
    return out
