"""Pins for the attention oracle.

Each check fixes the oracle against something other than itself: brute force,
a library routine (torch SDPA in fp64 with an explicit mask), closed forms,
a planted needle, the LSE-merge identity and sharing invariance."""
import math

import numpy as np
import pytest
import torch

from oracle import attention as A
from oracle import tree as T
from synth import values as V
from tests.helpers import random_workload

HEADS = [(1, 1), (2, 1), (4, 2), (8, 1)]


def _rand(rng, n, hq, hkv, d, q):
    K = rng.integers(-128, 128, size=(n, hkv, d)) / 128.0
    Vv = rng.integers(-128, 128, size=(n, hkv, d)) / 128.0
    Q = rng.integers(-128, 128, size=(q, hq, d)) / 128.0
    return K, Vv, Q


@pytest.mark.parametrize("seed", range(6))
def test_bruteforce_matches(seed):
    rng = np.random.default_rng(seed)
    hq, hkv = HEADS[seed % 4]
    d = 64 if seed % 2 else 16
    n = int(rng.integers(1, 20))
    q = int(rng.integers(1, n + 1))
    K, Vv, Q = _rand(rng, n, hq, hkv, d, q)
    O, lse = A.attention_request(K, Vv, Q, q)
    Ob, lseb = A.attention_bruteforce(K, Vv, Q, q)
    assert np.max(np.abs(O - Ob)) < 1e-12
    assert np.max(np.abs(lse - lseb)) < 1e-12


@pytest.mark.parametrize("seed", range(4))
def test_torch_sdpa_fp64(seed):
    rng = np.random.default_rng(100 + seed)
    hq, hkv = HEADS[seed]
    d = 128 if seed % 2 else 64
    n, q = 37, 9
    K, Vv, Q = _rand(rng, n, hq, hkv, d, q)
    O, _ = A.attention_request(K, Vv, Q, q)
    g = hq // hkv
    Kt = torch.tensor(K).permute(1, 0, 2).repeat_interleave(g, 0)        # [Hq, n, d]
    Vt = torch.tensor(Vv).permute(1, 0, 2).repeat_interleave(g, 0)
    Qt = torch.tensor(Q).permute(1, 0, 2)                                # [Hq, q, d]
    pos = torch.arange(n - q, n)
    mask = torch.arange(n)[None, :] <= pos[:, None]
    Ot = torch.nn.functional.scaled_dot_product_attention(Qt, Kt, Vt, attn_mask=mask)
    assert np.max(np.abs(Ot.permute(1, 0, 2).numpy() - O)) < 1e-12


def test_closed_forms():
    rng = np.random.default_rng(7)
    K, Vv, Q = _rand(rng, 5, 2, 1, 64, 5)
    # single visible key: query at position 0 sees only key 0
    O, lse = A.attention_request(K[:1], Vv[:1], Q[:1], 1)
    assert np.allclose(O[0, :], Vv[0, 0][None, :], atol=0, rtol=0)
    s0 = Q[0] @ K[0, 0] / math.sqrt(64)
    assert np.allclose(lse[0], s0, atol=1e-14)
    # all keys identical -> mean of visible V
    Ki = np.repeat(K[:1], 5, axis=0)
    O, _ = A.attention_request(Ki, Vv, Q, 5)
    for t in range(5):
        assert np.allclose(O[t], Vv[:t + 1, 0].mean(axis=0)[None, :], atol=1e-14)
    # Q = 0 -> mean of visible V and lse = ln(j+1)
    O, lse = A.attention_request(K, Vv, np.zeros_like(Q), 5)
    for t in range(5):
        assert np.allclose(O[t], Vv[:t + 1, 0].mean(axis=0)[None, :], atol=1e-14)
        assert np.allclose(lse[t], math.log(t + 1), atol=1e-14)


def test_planted_needle():
    rng = np.random.default_rng(9)
    n, d = 1000, 128
    K, Vv, Q = _rand(rng, n, 4, 1, d, 1)
    needle = 417
    Q[0, 2] = 8.0 * K[needle, 0]
    O, _ = A.attention_request(K, Vv, Q, 1)
    assert np.max(np.abs(O[0, 2] - Vv[needle, 0])) < 1e-6
    assert np.max(np.abs(O[0, 0] - Vv[needle, 0])) > 1e-2      # other heads unaffected


def test_future_keys_do_not_matter():
    rng = np.random.default_rng(3)
    K, Vv, Q = _rand(rng, 30, 4, 2, 64, 10)
    O, lse = A.attention_request(K, Vv, Q, 10)
    K2, V2 = K.copy(), Vv.copy()
    K2[25:] = 5.0
    V2[25:] = -7.0
    O2, lse2 = A.attention_request(K2, V2, Q, 10)
    assert np.array_equal(O[:5], O2[:5]) and np.array_equal(lse[:5], lse2[:5])
    assert not np.allclose(O[5:], O2[5:])


@pytest.mark.parametrize("seed", range(5))
def test_lse_merge_identity(seed):
    rng = np.random.default_rng(50 + seed)
    hq, hkv = HEADS[seed % 4]
    n, q = 60, 7
    K, Vv, Q = _rand(rng, n, hq, hkv, 64, q)
    qpos = np.arange(n - q, n)
    full = A.partial(K, Vv, Q, qpos, np.arange(n))
    ref = A.attention_request(K, Vv, Q, q)
    assert np.max(np.abs(full[0] - ref[0])) < 1e-12
    cuts = np.sort(rng.choice(np.arange(1, n), size=int(rng.integers(1, 6)), replace=False))
    bounds = [0, *cuts.tolist(), n]
    parts = []
    for a, b in zip(bounds[:-1], bounds[1:]):
        idx = np.arange(a, b)
        parts.append(A.partial(K[idx], Vv[idx], Q, qpos, idx))
    # a range beyond every query (fully masked) contributes weight 0
    parts.append((np.full_like(full[0], 123.0), np.full_like(full[1], -np.inf)))
    O, L = A.lse_merge(parts)
    assert np.max(np.abs(O - ref[0])) < 1e-12
    assert np.max(np.abs(L - ref[1])) < 1e-12


@pytest.mark.parametrize("seed", range(12))
def test_sharing_invariance(seed):
    """Node-wise cascade over the oracle tree (each path node attended once as
    its own partial, merged by LSE) == the per-request unshared definition."""
    hq, hkv = HEADS[seed % 4]
    w = random_workload(seed, hq=hq, hkv=hkv, d=64 if seed % 2 else 128)
    view = T.build(w, min_sep_len=0)
    for r in range(w.n_req):
        K, Vv, Q = A.request_inputs(w, r)
        q = int(w.q_len[r])
        n = K.shape[0]
        qpos = np.arange(n - q, n)
        parts = []
        for k in range(int(view["req_path_off"][r]), int(view["req_path_off"][r + 1])):
            nd = int(view["req_path_nodes"][k])
            s, ln = int(view["node_start"][nd]), int(view["node_len"][nd])
            idx = np.arange(s, s + ln)
            parts.append(A.partial(K[idx], Vv[idx], Q, qpos, idx))
        O, L = A.lse_merge(parts)
        Oref, Lref = A.attention_request(K, Vv, Q, q)
        assert np.max(np.abs(O - Oref)) < 1e-12
        assert np.max(np.abs(L - Lref)) < 1e-12


def test_workload_inputs_use_generator():
    w = random_workload(3, hq=2, hkv=1, d=64)
    K, Vv, Q = A.request_inputs(w, 0)
    K2, V2 = V.path_kv(w.path(0), w.seed, 1, 64)
    assert np.array_equal(K, K2) and np.array_equal(Vv, V2)
