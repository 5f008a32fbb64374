"""Data-parallel (subtree-sharded) and head-parallel plumbing shared by bench.py and the
multi-process tests (PAPER §7.1).

Data parallelism (strong scaling of ONE global batch): every rank builds the global
tree through the C ABI, blend_shard splits the density-sorted request order into 2N
weight-balanced blocks with subtree-snapped cuts and pairs block g with block 2N-1-g
("split continuous requests from both sides of the prefix tree"); each rank
builds, fills and runs only its shard — no KV crosses GPUs.  Afterwards the outputs
and LSE rows are all-gathered over the process group (NCCL over NVLink on the GPU
box, gloo in the CPU tests) and re-assembled in global request order by req_shard.

Head parallelism (NEXT-4): rank k of N takes kv heads [k Hkv/N, (k+1) Hkv/N)
and their query-head groups for the whole batch (an ordinary plan over Hq/N, Hkv/N
heads); the synthetic values keep GLOBAL head indices (head0 / kv_head0 offsets of
the fillers), so the N slices concatenated along the head axis are the full-head
problem; outputs are all-gathered along heads.

Input plumbing and collectives only; the method's arithmetic runs in libblend.
"""
from __future__ import annotations

import time

import numpy as np

from harness.run import build_tree, subset


def shard_batch(gw, world: int, rank: int, tree_kw=None, kappa: int = 213):
    """(local workload, req_shard int32[R], host seconds) of rank `rank` of `world`."""
    t0 = time.perf_counter()
    if world == 1:
        return gw, np.zeros(gw.n_req, dtype=np.int32), 0.0
    gtree = build_tree(gw, **(tree_kw or {}))
    req_shard, _ = gtree.shard(world, kappa)
    mine = np.nonzero(req_shard == rank)[0]
    w = subset(gw, mine, name=f"{gw.name}_shard{rank}of{world}")
    return w, req_shard, time.perf_counter() - t0


def row_index(gw, req_shard, world: int):
    """For each rank g, the global q rows (caller request order of the global batch) of
    its local rows, in its local order (its requests ascending, each request's q rows)."""
    qo = np.concatenate([[0], np.cumsum(gw.q_len.astype(np.int64))])
    out = []
    for g in range(world):
        rs = np.nonzero(req_shard == g)[0]
        out.append(np.concatenate([np.arange(qo[r], qo[r + 1]) for r in rs]) if len(rs)
                   else np.zeros(0, dtype=np.int64))
    return out


def gather_rows(out, lse, gw, req_shard, world: int, dist, dst=0):
    """All-gather every rank's (out [T_g, Hq, D], lse [T_g, Hq]) and, on rank `dst`,
    scatter them into global request order.  Returns (out_full, lse_full) on dst, else
    (None, None).  Works for any torch device the process group supports."""
    import torch
    rows = torch.tensor([out.shape[0]], dtype=torch.int64, device=out.device)
    dist.all_reduce(rows, op=dist.ReduceOp.MAX)
    R = int(rows.item())
    po = torch.zeros((R,) + tuple(out.shape[1:]), dtype=out.dtype, device=out.device)
    pl = torch.zeros((R,) + tuple(lse.shape[1:]), dtype=lse.dtype, device=lse.device)
    po[:out.shape[0]] = out
    pl[:lse.shape[0]] = lse
    go = [torch.empty_like(po) for _ in range(world)]
    gl = [torch.empty_like(pl) for _ in range(world)]
    dist.all_gather(go, po)
    dist.all_gather(gl, pl)
    if dist.get_rank() != dst:
        return None, None
    idx = row_index(gw, req_shard, world)
    T = int(gw.q_len.sum())
    of = torch.empty((T,) + tuple(out.shape[1:]), dtype=out.dtype, device=out.device)
    lf = torch.empty((T,) + tuple(lse.shape[1:]), dtype=lse.dtype, device=lse.device)
    seen = torch.zeros(T, dtype=torch.int32, device=out.device)
    for g in range(world):
        ix = torch.from_numpy(idx[g]).to(out.device)
        n = ix.numel()
        of.index_copy_(0, ix, go[g][:n])
        lf.index_copy_(0, ix, gl[g][:n])
        seen.index_add_(0, ix, torch.ones(n, dtype=torch.int32, device=out.device))
    assert bool((seen == 1).all()), "a global row was produced by zero or several ranks"
    return of, lf


def tp_heads(gw, world: int, rank: int):
    """Head slice of rank `rank` (NEXT-4): (Hq/N, Hkv/N, q head0, kv head0)."""
    if gw.num_kv_heads % world:
        raise ValueError(f"{gw.num_kv_heads} kv heads do not split over {world} ranks")
    hkv = gw.num_kv_heads // world
    hq = gw.num_q_heads // world
    return hq, hkv, rank * hq, rank * hkv


def gather_heads(out, lse, world: int, dist, dst=0):
    """All-gather head slices (out [T, Hq/N, D], lse [T, Hq/N]) into [T, Hq, D], [T, Hq]."""
    import torch
    go = [torch.empty_like(out) for _ in range(world)]
    gl = [torch.empty_like(lse) for _ in range(world)]
    dist.all_gather(go, out)
    dist.all_gather(gl, lse)
    if dist.get_rank() != dst:
        return None, None
    return torch.cat(go, dim=1), torch.cat(gl, dim=1)
