"""Attention oracle — fp64, per request, over the request's full materialised path.

TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).  Never used by the product.

What it computes; the paper never writes the attention math
out, so this is the textbook definition (Vaswani et al., cited at PAPER P:54):

  * decode "conditioned on all previous tokens" and each decode step
    "loads all p+i tokens": query at absolute position j sees keys
    i = 0..j of its own path (reading #3: key visible iff key_pos <= query_pos);
  * the root->leaf path is the request's prefix, so the oracle needs no
    tree: prefix sharing and cascade reuse must not change
    the result;
  * scale 1/sqrt(D) (reading #1); GQA kvh = h // (Hq/Hkv) (reading #2);
  * lse is the natural-log log-sum-exp of the scaled scores (reading #16).

For request r, query t (position j = n_r - q_r + t) and q head h:
    s_i = Q[t,h] . K[i,kvh] / sqrt(D)        i = 0..j
    m = max s,  w_i = exp(s_i - m),  l = sum w
    O = sum w_i V[i,kvh] / l,   lse = m + ln l
"""
from __future__ import annotations

import math
from typing import Dict, Iterable, Optional, Tuple

import numpy as np

from synth import values as V


def attention_request(K: np.ndarray, Vv: np.ndarray, Q: np.ndarray, q_len: int):
    """fp64 causal GQA attention of the last q_len path positions.

    K, Vv: [n, Hkv, D] (the request's full path); Q: [q_len, Hq, D].
    Returns O [q_len, Hq, D], lse [q_len, Hq] (float64).
    """
    K = np.asarray(K, dtype=np.float64)
    Vv = np.asarray(Vv, dtype=np.float64)
    Q = np.asarray(Q, dtype=np.float64)
    n, hkv, d = K.shape
    hq = Q.shape[1]
    g = hq // hkv
    Qg = Q.reshape(q_len, hkv, g, d)
    # scores [q, Hkv, g, n]
    s = np.einsum("tkgd,nkd->tkgn", Qg, K) / math.sqrt(d)
    pos_q = n - q_len + np.arange(q_len)
    visible = np.arange(n)[None, :] <= pos_q[:, None]          # [q, n]
    s = np.where(visible[:, None, None, :], s, -np.inf)
    m = s.max(axis=-1, keepdims=True)
    w = np.exp(s - m)
    l = w.sum(axis=-1, keepdims=True)
    O = np.einsum("tkgn,nkd->tkgd", w, Vv) / l
    lse = (m + np.log(l))[..., 0]
    return O.reshape(q_len, hq, d), lse.reshape(q_len, hq)


def attention_bruteforce(K, Vv, Q, q_len):
    """Same definition with Python loops and math.fsum (tiny inputs only)."""
    n, hkv, d = K.shape
    hq = Q.shape[1]
    g = hq // hkv
    O = np.zeros((q_len, hq, d))
    lse = np.zeros((q_len, hq))
    for t in range(q_len):
        j = n - q_len + t
        for h in range(hq):
            kvh = h // g
            s = [math.fsum(float(Q[t, h, e]) * float(K[i, kvh, e]) for e in range(d)) / math.sqrt(d)
                 for i in range(j + 1)]
            m = max(s)
            w = [math.exp(x - m) for x in s]
            l = math.fsum(w)
            for e in range(d):
                O[t, h, e] = math.fsum(w[i] * float(Vv[i, kvh, e]) for i in range(j + 1)) / l
            lse[t, h] = m + math.log(l)
    return O, lse


def request_inputs(w, r: int):
    """Materialise (K, V, Q) of request r from the synthetic generator (fp64,
    exactly the bf16/fp32 grid values the device sees)."""
    path = w.path(r)
    K, Vv = V.path_kv(path, w.seed, w.num_kv_heads, w.head_dim, w.kv_head0)
    q = int(w.q_len[r])
    Q = V.q_values(w.gid(r), np.arange(q), w.seed, w.num_q_heads, w.head_dim, w.scale_q, w.head0)
    return K, Vv, Q


def attention_workload(w, requests: Optional[Iterable[int]] = None) -> Dict[int, Tuple[np.ndarray, np.ndarray]]:
    """{r: (O [q_r,Hq,D], lse [q_r,Hq])} for the requested request indices."""
    out = {}
    for r in (range(w.n_req) if requests is None else requests):
        K, Vv, Q = request_inputs(w, r)
        out[int(r)] = attention_request(K, Vv, Q, int(w.q_len[r]))
    return out


def partial(K, Vv, Q, q_pos, k_pos):
    """Attention of queries (absolute positions q_pos) restricted to the keys at
    absolute positions k_pos (a subset of the path).  Returns (O, lse); rows with
    no visible key get O = 0, lse = -inf (reading #16)."""
    n, hkv, d = K.shape
    hq = Q.shape[1]
    g = hq // hkv
    qn = Q.shape[0]
    Qg = Q.reshape(qn, hkv, g, d)
    s = np.einsum("tkgd,nkd->tkgn", Qg, K) / math.sqrt(d)
    vis = np.asarray(k_pos)[None, :] <= np.asarray(q_pos)[:, None]
    s = np.where(vis[:, None, None, :], s, -np.inf)
    m = s.max(axis=-1, keepdims=True) if s.shape[-1] else np.full(s.shape[:-1] + (1,), -np.inf)
    m_safe = np.where(np.isfinite(m), m, 0.0)
    w_ = np.exp(s - m_safe) if s.shape[-1] else s
    l = w_.sum(axis=-1, keepdims=True)
    O = np.where(l > 0, np.einsum("tkgn,nkd->tkgd", w_, Vv) / np.where(l > 0, l, 1.0), 0.0)
    lse = np.where(l[..., 0] > 0, (m_safe + np.log(np.where(l > 0, l, 1.0)))[..., 0], -np.inf)
    return O.reshape(qn, hq, d), lse.reshape(qn, hq)


def lse_merge(parts):
    """Merge partial (O_i, lse_i) by log-sum-exp (reading #16/#17):
    L = max lse_i + ln sum exp(lse_i - max), O = sum exp(lse_i - L) O_i.
    -inf partials carry weight 0; all -inf -> (0, -inf)."""
    lses = np.stack([p[1] for p in parts])          # [k, q, h]
    Os = np.stack([p[0] for p in parts])            # [k, q, h, d]
    mx = lses.max(axis=0)
    mx_safe = np.where(np.isfinite(mx), mx, 0.0)
    w = np.exp(lses - mx_safe[None])
    tot = w.sum(axis=0)
    L = np.where(tot > 0, mx_safe + np.log(np.where(tot > 0, tot, 1.0)), -np.inf)
    wn = np.where(tot[None] > 0, w / np.where(tot > 0, tot, 1.0)[None], 0.0)
    O = (wn[..., None] * Os).sum(axis=0)
    return O, L
