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
               free_pages=None):
    fp = w.free_pages if free_pages is None else free_pages
    return B.build(w.tokens, w.tok_off, w.q_len, w.prompt_len, w.out_len,
                   num_q_heads=w.num_q_heads, num_kv_heads=w.num_kv_heads, head_dim=w.head_dim,
                   kv_dtype=w.kv_dtype, model_params=w.model_params, hidden=w.hidden, layers=w.layers,
                   page_size=w.page_size, free_pages=fp, global_id=w.global_id, rows_min=rows_min,
                   min_sep_len=min_sep_len, force_class=force_class, split_tokens=split_tokens,
                   num_sms=num_sms)


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

    def run(self, path=B.PATH_AUTO, stream=None, events=None):
        B.attention(self.q, self.k_cache, self.v_cache, self.plan, self.out, self.lse, self.ws,
                    n_cache_pages=self.n_cache_pages, path=path, stream=stream, events=events)


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
                  torch.from_numpy(phash.view(np.int64)).to(device), w.seed)
        gid, tt = query_rows(w)
        B.fill_q(q, w.kv_dtype, w.num_q_heads, w.head_dim, torch.from_numpy(gid).to(device),
                 torch.from_numpy(tt).to(device), w.seed, w.scale_q)
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
