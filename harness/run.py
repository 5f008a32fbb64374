"""Workload -> libblend: tree build, page hashes, device buffers, fills, attention.

Input plumbing only: the method's arithmetic runs in libblend (device) and, for
checking, in oracle/ (CPU).  This module never imports oracle/.
"""
from __future__ import annotations

import time
from dataclasses import dataclass
from typing import Optional

import numpy as np

import paper_2411_16102_b200 as B
from synth import values as V


def build_tree(w, rows_min=128, min_sep_len=128, force_class=0, split_tokens=0, num_sms=148,
               free_pages=None, dense_split=0, split_waste=0):
    fp = w.free_pages if free_pages is None else free_pages
    return B.build(w.tokens, w.tok_off, w.q_len, w.prompt_len, w.out_len,
                   num_q_heads=w.num_q_heads, num_kv_heads=w.num_kv_heads, head_dim=w.head_dim,
                   kv_dtype=w.kv_dtype, model_params=w.model_params, hidden=w.hidden, layers=w.layers,
                   page_size=w.page_size, free_pages=fp, global_id=w.global_id, rows_min=rows_min,
                   min_sep_len=min_sep_len, force_class=force_class, split_tokens=split_tokens,
                   num_sms=num_sms, dense_split=dense_split, split_waste=split_waste)


def page_slot_hashes(w, view):
    """(page_ids int32[P], page_count int32[P], page_hash uint64[P*ps]) for every page
    the tree uses: slot s of page k of node N holds position start(N) + k*ps + s."""
    ps = w.page_size
    N = view["n_nodes"]
    P = int(view["node_page_off"][-1])
    page_count = np.zeros(P, dtype=np.int32)
    page_hash = np.zeros(P * ps, dtype=np.uint64)
    h_end = np.zeros(N, dtype=np.uint64)
    for i in range(N):                       # parents precede children (preorder ids)
        s, ln = int(view["node_start"][i]), int(view["node_len"][i])
        par = int(view["node_parent"][i])
        hp = int(h_end[par]) if par >= 0 else 0
        r0 = int(view["node_first_req"][i])
        toks = w.tokens[w.tok_off[r0] + s: w.tok_off[r0] + s + ln]
        h = V.segment_hash(toks, s, hp, w.seed)
        h_end[i] = h[-1]
        p0 = int(view["node_page_off"][i])
        npg = int(view["node_page_off"][i + 1]) - p0
        page_count[p0:p0 + npg] = np.minimum(ps, ln - ps * np.arange(npg))
        buf = np.zeros(npg * ps, dtype=np.uint64)
        buf[:ln] = h
        page_hash[p0 * ps:(p0 + npg) * ps] = buf
    return view["page_table"].astype(np.int32), page_count, page_hash


def query_rows(w):
    """(row_gid int64[T], row_t int32[T]) of q rows in caller request order."""
    gid = np.repeat(np.asarray([w.gid(r) for r in range(w.n_req)], dtype=np.int64), w.q_len)
    t = np.concatenate([np.arange(int(q), dtype=np.int32) for q in w.q_len])
    return gid, t


@dataclass
class DeviceBatch:
    w: object
    tree: object
    view: dict
    plan: object
    q: object
    k_cache: object
    v_cache: object
    out: object
    lse: object
    ws: object
    n_cache_pages: int
    build_s: float
    info: dict

    def run(self, path=B.PATH_AUTO, stream=None, events=None, flags=0):
        B.attention(self.q, self.k_cache, self.v_cache, self.plan, self.out, self.lse, self.ws,
                    n_cache_pages=self.n_cache_pages, path=path, stream=stream, events=events,
                    flags=flags)


def device_batch(w, device="cuda", tree_kw=None, n_cache_pages=None, fill=True) -> DeviceBatch:
    import torch
    tree_kw = tree_kw or {}
    t0 = time.perf_counter()
    tree = build_tree(w, **tree_kw)
    build_s = time.perf_counter() - t0
    view = tree.view()
    dt = torch.bfloat16 if w.kv_dtype == "bf16" else torch.float32
    P = int(view["n_pages"])
    maxpage = int(view["page_table"].max()) + 1 if P else 1
    ncp = max(maxpage, n_cache_pages or 0)
    T = w.sum_q
    k_cache = torch.zeros((ncp, w.num_kv_heads, w.page_size, w.head_dim), dtype=dt, device=device)
    v_cache = torch.zeros_like(k_cache)
    q = torch.zeros((T, w.num_q_heads, w.head_dim), dtype=dt, device=device)
    out = torch.zeros_like(q)
    lse = torch.zeros((T, w.num_q_heads), dtype=torch.float32, device=device)
    ws = torch.empty(max(256, tree.workspace_bytes), dtype=torch.uint8, device=device)
    plan_buf = torch.empty(max(256, tree.plan_bytes), dtype=torch.uint8, device=device)
    plan = tree.upload_plan(plan_buf)
    if fill:
        pid, pcnt, phash = page_slot_hashes(w, view)
        B.fill_kv(k_cache, v_cache, w.kv_dtype, w.num_kv_heads, w.head_dim, w.page_size,
                  torch.from_numpy(pid).to(device), torch.from_numpy(pcnt).to(device),
                  torch.from_numpy(phash.view(np.int64)).to(device), w.seed, kv_head0=w.kv_head0)
        gid, tt = query_rows(w)
        B.fill_q(q, w.kv_dtype, w.num_q_heads, w.head_dim, torch.from_numpy(gid).to(device),
                 torch.from_numpy(tt).to(device), w.seed, w.scale_q, head0=w.head0)
    torch.cuda.synchronize()
    return DeviceBatch(w, tree, view, plan, q, k_cache, v_cache, out, lse, ws, ncp, build_s,
                       tree.plan_info())


def work_counts(w, view):
    """Algorithmic work: F_alg = 4 D Hq sum(pos+1) over query tokens;
    B_alg = distinct KV bytes + Q read + O written."""
    n = np.diff(w.tok_off).astype(np.int64)
    q = w.q_len.astype(np.int64)
    spos = (q * (n - q) + q * (q + 1) // 2).sum()
    F = 4 * w.head_dim * w.num_q_heads * int(spos)
    b = 2 if w.kv_dtype == "bf16" else 4
    kv = int(view["node_len"].astype(np.int64).sum()) * w.num_kv_heads * w.head_dim * 2 * b
    qo = int(q.sum()) * w.num_q_heads * w.head_dim * b * 2
    return F, kv + qo, kv


def subset(w, reqs, name=None):
    """Workload restricted to requests `reqs` (ascending), keeping global ids."""
    from synth.workloads import Workload
    reqs = np.asarray(reqs, dtype=np.int64)
    paths = [w.path(int(r)) for r in reqs]
    tok_off = np.zeros(len(reqs) + 1, dtype=np.int64)
    if len(reqs):
        tok_off[1:] = np.cumsum([len(p) for p in paths])
    gid = np.asarray([w.gid(int(r)) for r in reqs], dtype=np.int64)
    return Workload(name=name or w.name, seed=w.seed, num_q_heads=w.num_q_heads,
                    num_kv_heads=w.num_kv_heads, head_dim=w.head_dim, kv_dtype=w.kv_dtype,
                    page_size=w.page_size, model_params=w.model_params, hidden=w.hidden,
                    layers=w.layers,
                    tokens=np.concatenate(paths).astype(np.int32) if paths else np.zeros(0, np.int32),
                    tok_off=tok_off, q_len=w.q_len[reqs], prompt_len=w.prompt_len[reqs],
                    out_len=w.out_len[reqs], scale_q=w.scale_q, global_id=gid, head0=w.head0,
                    kv_head0=w.kv_head0)


def pass_work(w, view, rows_min=128, force_class=0):
    """Algorithmic work of the two passes, mirroring the planner's item split:
    SEPARATE-node items and BIG-request items are dense iff rows*g >= rows_min.
    Returns dict(dense_flops, dense_bytes, stream_flops, stream_bytes) where
    flops = 4 D x (visible (row, key) pairs) and bytes = distinct KV bytes of the
    pass's items + Q read + O written (dtype bytes)."""
    g = w.num_q_heads // w.num_kv_heads
    D, Hq, Hkv = w.head_dim, w.num_q_heads, w.num_kv_heads
    b = 2 if w.kv_dtype == "bf16" else 4
    n = np.diff(w.tok_off)
    ncls, rcls = view["node_class"], view["req_class"]
    start, ln = view["node_start"], view["node_len"]
    po, pn = view["req_path_off"], view["req_path_nodes"]

    def vis(r, node):
        a = int(n[r]) - int(w.q_len[r])
        pos = np.arange(a, int(n[r]))
        return int(np.clip(pos - int(start[node]) + 1, 0, int(ln[node])).sum())

    sep_rows = {}
    sep_vis = {}
    out = dict(dense_flops=0, dense_bytes=0, stream_flops=0, stream_bytes=0)
    for r in range(w.n_req):
        folded_vis, folded_len = 0, 0
        for k in range(int(po[r]), int(po[r + 1])):
            node = int(pn[k])
            if ncls[node] and (not rcls[r] or force_class == 1):
                sep_rows[node] = sep_rows.get(node, 0) + int(w.q_len[r])
                sep_vis[node] = sep_vis.get(node, 0) + vis(r, node)
            else:
                folded_vis += vis(r, node)
                folded_len += int(ln[node])
        if folded_len == 0:
            continue
        dense = int(w.q_len[r]) * g >= rows_min
        key = "dense" if dense else "stream"
        out[key + "_flops"] += 4 * D * Hq * folded_vis
        out[key + "_bytes"] += folded_len * Hkv * D * 2 * b + 2 * int(w.q_len[r]) * Hq * D * b
    for node, rows in sep_rows.items():
        key = "dense" if rows * g >= rows_min else "stream"
        out[key + "_flops"] += 4 * D * Hq * sep_vis[node]
        out[key + "_bytes"] += int(ln[node]) * Hkv * D * 2 * b + 2 * rows * Hq * D * b
    return out
