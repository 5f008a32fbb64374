"""Pins for the descriptor oracle.

Pinned to: SPEC worked examples, the literal
definition of a node (maximal run of constant A(pi)) by brute force, the
paper's cost model for single requests, the paper's density
statements, invariances and rejections."""
from fractions import Fraction

import numpy as np
import pytest

from oracle import tree as T
from synth import workloads as W
from tests.helpers import from_paths, random_workload

A100_TF, A100_BW = 312e12, 2039e9      # A100 80GB SXM peak fp16 / bandwidth


def _node_tokens(v, w, i):
    s, ln = int(v["node_start"][i]), int(v["node_len"][i])
    return tuple(int(x) for x in w.path(int(v["node_first_req"][i]))[s:s + ln])


def _shape(v, w):
    """Canonical tree shape independent of ids: {(path-of-token-tuples, ends)}"""
    out = set()
    for i in range(v["n_nodes"]):
        chain, x = [], i
        while x >= 0:
            chain.append(_node_tokens(v, w, x))
            x = int(v["node_parent"][x])
        out.add((tuple(reversed(chain)), int(v["node_nreq"][i])))
    return out


def test_spec_ab_ac():
    # S:155 requests "AB","AC" -> root segment "A" with two leaf children "B","C"
    A_, B_, C_ = 1001, 1002, 1003
    w = from_paths([[A_, B_], [A_, C_]])
    v = T.build(w)
    assert v["n_nodes"] == 3
    assert _node_tokens(v, w, 0) == (A_,) and int(v["node_parent"][0]) == -1
    kids = {_node_tokens(v, w, i) for i in (1, 2)}
    assert kids == {(B_,), (C_,)}
    assert all(int(v["node_parent"][i]) == 0 for i in (1, 2))


def test_spec_identical_prompts_share_leaf():
    # S:154 two identical prompts -> one leaf holding both ids
    w = from_paths([[5000, 5001, 5002], [5000, 5001, 5002]])
    v = T.build(w)
    assert v["n_nodes"] == 1 and v["node_ends"][0] == [0, 1]


def test_prefix_request_ends_node():
    # "ABC","AB" -> "AB" with child "C" (a request end is a node boundary)
    w = from_paths([[7, 8, 9], [7, 8]])
    v = T.build(w)
    assert v["n_nodes"] == 2 and _node_tokens(v, w, 0) == (7, 8) and _node_tokens(v, w, 1) == (9,)
    assert v["node_ends"][0] == [1] and v["node_ends"][1] == [0]


@pytest.mark.parametrize("N", [2, 5, 17])
def test_spec_common_prompt_shared_tokens(N):
    # S:156 N requests with a common 100-token prompt: shared tokens = 100 (N-1)
    rng = np.random.default_rng(N)
    sysp = rng.integers(1000, 32000, 100)
    paths = [np.concatenate([sysp, [40000 + i], rng.integers(1000, 32000, int(rng.integers(0, 9)))])
             for i in range(N)]
    w = from_paths(paths)
    v = T.build(w)
    assert int(np.diff(w.tok_off).sum()) - int(v["node_len"].sum()) == 100 * (N - 1)


def _bruteforce_nodes(w):
    """Literal definition: along each path, a new node starts at j+1 iff
    A(pi_{j+1}) != A(pi_j), A(pi) = {requests having prefix pi}."""
    paths = [tuple(int(t) for t in w.path(r)) for r in range(w.n_req)]
    def A(pref):
        return frozenset(r for r, p in enumerate(paths) if len(p) >= len(pref) and p[:len(pref)] == pref)
    nodes = set()
    for p in paths:
        start = 0
        for j in range(1, len(p) + 1):
            if j == len(p) or A(p[:j + 1]) != A(p[:j]):
                nodes.add((p[:start], p[start:j]))
                start = j
    return nodes


@pytest.mark.parametrize("seed", range(25))
def test_trie_matches_literal_definition(seed):
    w = random_workload(seed, tok_lo=1000, tok_hi=1004 if seed % 3 == 0 else 32000, max_seg=12)
    v = T.build(w)
    got = set()
    for i in range(v["n_nodes"]):
        s = int(v["node_start"][i])
        full = tuple(int(t) for t in w.path(int(v["node_first_req"][i]))[:s + int(v["node_len"][i])])
        got.add((full[:s], full[s:]))
    assert got == _bruteforce_nodes(w)
    # every request's path nodes concatenate to its tokens
    for r in range(w.n_req):
        toks = []
        for k in range(int(v["req_path_off"][r]), int(v["req_path_off"][r + 1])):
            toks.extend(_node_tokens(v, w, int(v["req_path_nodes"][k])))
        assert tuple(toks) == tuple(int(t) for t in w.path(r))


@pytest.mark.parametrize("seed", range(10))
def test_insertion_order_independent(seed):
    # S:151 / S:225
    w = random_workload(seed)
    perm = np.random.default_rng(seed).permutation(w.n_req)
    w2 = from_paths([w.path(int(r)) for r in perm], q=w.q_len[perm], p=w.prompt_len[perm],
                    d=w.out_len[perm])
    assert _shape(T.build(w), w) == _shape(T.build(w2), w2)


def _comp_mem_single(p, d, Pm=8_030_261_248, H=4096, L=32):
    """Paper cost model, P:89 and P:93 (exact sum form), hardware constants removed."""
    comp = (p + d) * Pm * 2 + p * p * H * L * 4
    mem = sum(p + i for i in range(1, d + 1))
    return comp, mem


@pytest.mark.parametrize("p,d", [(1, 0), (64, 16), (728, 256), (228, 16384), (1100, 2), (3000, 4000)])
def test_single_request_key_is_paper_cost(p, d):
    w = from_paths([list(range(1000, 1000 + p))], p=[p], d=[d])
    v = T.build(w)
    comp, mem = _comp_mem_single(p, d)
    assert v["cu"][0] == comp and v["mu"][0] == mem


def test_shared_prompt_counted_once():
    # two identical-prompt requests: t_comp counts the prompt once plus two decode streams
    p, d1, d2 = 500, 30, 70
    w = from_paths([list(range(2000, 2000 + p))] * 2, p=[p, p], d=[d1, d2])
    v = T.build(w)
    Pm, H, L = 8_030_261_248, 4096, 32
    assert v["cu"][0] == 2 * Pm * (p + d1 + d2) + 4 * H * L * 2 * p * p
    assert v["mu"][0] == _comp_mem_single(p, d1)[1] + _comp_mem_single(p, d2)[1]


def _rho(cu, mu, compute=A100_TF, bw=A100_BW, hkv_total=1024, L=32):
    return (cu / compute) / (mu * hkv_total * L * 4 / bw)


def test_density_paper_statements():
    # P:106 ">4K output => memory-intensive" and P:328 MMLU (d=2) compute-intensive
    for p in (64, 256, 1024):
        cu, mu = _comp_mem_single(p, 4096)
        assert _rho(cu, mu) < 1
        cu, mu = _comp_mem_single(p, 2)
        assert _rho(cu, mu) > 1
    # P:379 worked example: densities 3.73 and 0.096 for BurstGPT-like / OpenVid-like nodes
    cu, mu = _comp_mem_single(728, 256)
    assert abs(_rho(cu, mu) / 3.73 - 1) < 0.02
    cu, mu = _comp_mem_single(228, 16384)
    assert abs(_rho(cu, mu) / 0.096 - 1) < 0.02


def test_kv_bytes_per_token_reading():
    # P:383 "one A100 80GB can hold nearly 500K tokens for an Llama-3.1-8B" with
    # H_kv L 4 = 1024*32*4 bytes per token (reading #8)
    per_tok = 1024 * 32 * 4
    assert per_tok == 131072
    assert 450_000 < (80 - 16) * 2**30 / per_tok < 550_000


def test_partition_worked_example():
    # rho 3.73 and 0.096, target 1.27, M = 60 GB -> 19.3 / 40.7 GB
    rl, rr, rt, M = 3.73, 0.096, 1.27, 60.0
    ml = M * (rt - rr) / (rl - rr)
    assert abs(ml - 19.3) < 0.1 and abs(M - ml - 40.7) < 0.1


def test_sort_example_spec():
    # S:181 children with rho [0.5, 3.0, 1.0] -> order [3.0, 1.0, 0.5]; the
    # densities are realised by single-request leaves of different d under one root
    sysp = list(range(3000, 3010))
    ds = [3000, 5, 200]                                  # rho low, high, mid
    paths = [sysp + [50000 + i] for i in range(3)]
    w = from_paths(paths, p=[11, 11, 11], d=ds)
    v = T.build(w)
    rhos = [Fraction(v["cu"][i], v["mu"][i]) for i in (1, 2, 3)]
    assert rhos == sorted(rhos, reverse=True)
    assert [v["node_ends"][i] for i in (1, 2, 3)] == [[1], [2], [0]]
    assert list(v["dfs_order"]) == [1, 2, 0]


def test_sort_is_fixed_point():
    # relabelling requests in DFS order and rebuilding yields the same order
    w = random_workload(5, n_req=12)
    v = T.build(w)
    order = v["dfs_order"]
    w2 = from_paths([w.path(int(r)) for r in order], q=w.q_len[order], p=w.prompt_len[order],
                    d=w.out_len[order])
    v2 = T.build(w2)
    assert list(v2["dfs_order"]) == list(range(w.n_req))


def test_ties_break_by_min_request_id():
    # S:232 identical densities -> smaller request id first
    paths = [[9000, 1], [9000, 2], [9000, 3]]
    w = from_paths(paths, p=[2, 2, 2], d=[5, 5, 5])
    v = T.build(w)
    assert list(v["dfs_order"]) == [0, 1, 2]
    w = from_paths(paths[::-1], p=[2, 2, 2], d=[5, 5, 5])
    assert list(T.build(w)["dfs_order"]) == [0, 1, 2]


def test_dfs_examples():
    # S:208 single chain -> the one request; "AB","AC","D" -> leaves in child order
    w = from_paths([[1, 2, 3]])
    assert list(T.build(w)["dfs_order"]) == [0]
    w = from_paths([[10, 11], [10, 12], [13]], p=[2, 2, 1], d=[1, 1, 1])
    v = T.build(w)
    assert sorted(v["dfs_order"]) == [0, 1, 2]
    # leaves appear in preorder node order
    leaf_order = [r for i in range(v["n_nodes"]) for r in v["node_ends"][i]]
    assert leaf_order == list(v["dfs_order"])


def test_zero_output_is_leftmost():
    # reading #13: MU = 0 means infinite density
    w = from_paths([[1, 2], [1, 3]], p=[2, 2], d=[100, 0])
    v = T.build(w)
    assert list(v["dfs_order"]) == [1, 0]


@pytest.mark.parametrize("seed", range(6))
def test_pages_and_paths(seed):
    w = random_workload(seed, page_size=16)
    free = np.random.default_rng(seed).permutation(5000).astype(np.int32)
    v = T.build(w, free_pages=free)
    need = [(int(x) + 15) // 16 for x in v["node_len"]]
    assert list(np.diff(v["node_page_off"])) == need
    assert np.array_equal(v["page_table"], free[:sum(need)])
    # preorder: parent id < child id, children consecutive subtrees
    for i in range(v["n_nodes"]):
        assert int(v["node_parent"][i]) < i


def test_classes_worked_cases():
    # C2: the 1024-token MMLU prefix is shared by 256 decode rows x g=4 >= 128 -> SEPARATE
    w = W.c2_mmlu_decode()
    v = T.build(w)
    big = [i for i in range(v["n_nodes"]) if v["node_len"][i] == 1024]
    assert len(big) == 1 and v["node_class"][big[0]] == 1 and int(v["node_class"].sum()) == 1
    assert int(v["req_class"].sum()) == 0
    # C1 mode c: the 64-token prompt is shorter than the 128-token cascade break-even
    w = W.c1_tiny("c")
    v = T.build(w)
    assert int(v["node_class"].sum()) == 0
    assert int(v["req_class"][8]) == 1            # q=64, g=2 -> 128 rows -> BIG
    v = T.build(w, min_sep_len=0)
    assert int(v["node_class"][0]) == 1
    v = T.build(w, force_class=2, min_sep_len=0)
    assert int(v["node_class"].sum()) == 0
    v = T.build(w, force_class=1)
    assert int(v["node_class"][0]) == 1
    # C3: 64 prefill chunks of 512 tokens x g=4 are BIG; video system prompt SEPARATE
    w = W.c3_burst_openvid()
    v = T.build(w)
    assert int(v["req_class"].sum()) == 64


@pytest.mark.parametrize("bad,status", [
    ("q0", T.EMALFORMED), ("qbig", T.EMALFORMED), ("empty", T.EMALFORMED), ("negtok", T.EMALFORMED),
    ("heads", T.EINVAL), ("dim", T.EUNSUPPORTED), ("ps", T.EINVAL), ("ps2", T.EINVAL),
    ("nospc", T.ENOSPC), ("dup", T.EINVAL),
])
def test_rejections(bad, status):
    kw = {}
    paths = [[1, 2, 3], [1, 2, 4]]
    q = [1, 1]
    w = from_paths(paths, q=q)
    if bad == "q0":
        w.q_len[0] = 0
    elif bad == "qbig":
        w.q_len[0] = 4
    elif bad == "empty":
        w = from_paths([[1, 2, 3], []], q=[1, 1])
    elif bad == "negtok":
        w.tokens[1] = -5
    elif bad == "heads":
        w.num_q_heads = 3; w.num_kv_heads = 2
    elif bad == "dim":
        w.head_dim = 96
    elif bad == "ps":
        w.page_size = 24
    elif bad == "ps2":
        w.page_size = 256
    elif bad == "nospc":
        kw["free_pages"] = np.array([0, 1], np.int32)
    elif bad == "dup":
        kw["free_pages"] = np.array([0, 1, 1, 3], np.int32)
    with pytest.raises(T.BlendError) as e:
        T.build(w, **kw)
    assert e.value.status == status


# ---------------------------------------------------------------------------
# Density key terms for requests whose cached path length n_r differs from the
# prompt length p_r (decode state n_r > p_r, chunked-prefill state n_r < p_r).
# Comp(r) counts (p + d) GEMM tokens and p^2 attention work of the WHOLE
# request, whatever step of its lifetime the snapshot catches; a set's
# GEMM tokens are (1 - s) T_comp, i.e. shared prompt tokens count once.
# ---------------------------------------------------------------------------
@pytest.mark.parametrize("p,d,n", [(64, 16, 1), (64, 16, 40), (64, 16, 64), (64, 16, 70), (64, 16, 80),
                                   (728, 256, 512), (728, 256, 900), (228, 16384, 5000), (1100, 2, 1101)])
def test_single_request_key_independent_of_lifetime_state(p, d, n):
    # n < p: prefill state (p - n prompt tokens not yet in the cache); n > p: decode
    # state (n - p generated tokens cached).  The key is the paper's Comp/Mem of the
    # request, independent of n.
    w = from_paths([list(range(1000, 1000 + n))], p=[p], d=[d])
    v = T.build(w)
    comp, mem = _comp_mem_single(p, d)
    assert v["cu"][0] == comp and v["mu"][0] == mem


def test_three_level_key_by_hand():
    # Worked by hand from P:89 (GEMM tokens = prompt + output) and P:315 (shared prompt
    # tokens counted once).  Tree: N0 (100 tokens, requests A B C) -> N1 (50, A B) ->
    # leaves a (10, A), b (20, B); N0 -> c (30, C).
    #   A: path 160 tokens, p = 120 (decode state: prompt = N0 + 20 tokens of N1)
    #   B: path 170 tokens, p = 200 (prefill state: 30 prompt tokens not yet cached)
    #   C: path 130 tokens, p = 130
    # Distinct prompt tokens of {A, B} = N0 100 + N1 50 (B's prompt covers it) + b 20 + B's
    # 30 uncached = 200; A's leaf holds generated tokens only.  Of {A, B, C}: 200 + c 30.
    rng = np.random.default_rng(7)
    n0, n1 = list(rng.integers(1000, 32000, 100)), [50000 + i for i in range(50)]
    a, b, c = [60000 + i for i in range(10)], [61000 + i for i in range(20)], [62000 + i for i in range(30)]
    dA, dB, dC = 50, 7, 300
    w = from_paths([n0 + n1 + a, n0 + n1 + b, n0 + c], p=[120, 200, 130], d=[dA, dB, dC])
    v = T.build(w)
    Pm, HL4 = 8_030_261_248, 4 * 4096 * 32

    def node_of(tokens):
        for i in range(v["n_nodes"]):
            if _node_tokens(v, w, i) == tuple(tokens):
                return i
        raise AssertionError(tokens)
    mem = lambda p, d: p * d + d * (d + 1) // 2          # noqa: E731  sum_{i=1..d} (p + i)
    expect = {
        tuple(n0): (230 + dA + dB + dC, [120, 200, 130], [(120, dA), (200, dB), (130, dC)]),
        tuple(n1): (200 + dA + dB, [120, 200], [(120, dA), (200, dB)]),
        tuple(a): (120 + dA, [120], [(120, dA)]),     # single request: G = p + d
        tuple(b): (200 + dB, [200], [(200, dB)]),
        tuple(c): (130 + dC, [130], [(130, dC)]),
    }
    for toks, (G, ps, pd) in expect.items():
        i = node_of(toks)
        assert v["cu"][i] == 2 * Pm * G + HL4 * sum(x * x for x in ps), toks[:2]
        assert v["mu"][i] == sum(mem(p, d) for p, d in pd)


def _bruteforce_key(w, S, Pm, HL4):
    """G_S = |distinct prompt tokens of S| + sum d_r, a prompt token being identified by
    its full prefix (tokens up to and including it) when it is cached, and as private
    (r, j) when it is not yet in the cache (j >= n_r)."""
    seen = set()
    for r in S:
        path = w.path(r)
        p, n = int(w.prompt_len[r]), len(path)
        for j in range(min(p, n)):
            seen.add(tuple(int(x) for x in path[:j + 1]))
        for j in range(n, p):
            seen.add(("uncached", r, j))
    G = len(seen) + sum(int(w.out_len[r]) for r in S)
    cu = 2 * Pm * G + HL4 * sum(int(w.prompt_len[r]) ** 2 for r in S)
    mu = sum(int(w.prompt_len[r]) * int(w.out_len[r]) + int(w.out_len[r]) * (int(w.out_len[r]) + 1) // 2
             for r in S)
    return cu, mu


@pytest.mark.parametrize("seed", range(12))
def test_keys_match_distinct_prompt_bruteforce(seed):
    # every node's key against the brute-force distinct-prefix count, with prompt lengths
    # drawn on both sides of the cached path length
    w = random_workload(seed, max_seg=15, tok_hi=1003 if seed % 4 == 0 else 32000)
    rng = np.random.default_rng(100 + seed)
    n = np.diff(w.tok_off)
    w.prompt_len = np.array([max(0, int(x) + int(rng.integers(-int(x), 12))) for x in n], dtype=np.int32)
    v = T.build(w)
    Pm, HL4 = int(w.model_params), 4 * int(w.hidden) * int(w.layers)
    for i in range(v["n_nodes"]):
        s, ln = int(v["node_start"][i]), int(v["node_len"][i])
        full = w.path(int(v["node_first_req"][i]))[:s + ln]
        S = [r for r in range(w.n_req) if len(w.path(r)) >= s + ln and np.array_equal(w.path(r)[:s + ln], full)]
        assert len(S) == int(v["node_nreq"][i])
        assert (v["cu"][i], v["mu"][i]) == _bruteforce_key(w, S, Pm, HL4), i


@pytest.mark.parametrize("p,d,n", [(64, 16, 40), (728, 256, 900), (228, 16384, 300), (1100, 2, 1101)])
def test_request_key_is_single_request_tree_key(p, d, n):
    w = from_paths([list(range(1000, 1000 + n))], p=[p], d=[d])
    v = T.build(w)
    assert T.request_key(p, d, 8_030_261_248, 4096, 32) == (v["cu"][0], v["mu"][0])
    # P:379 worked example with A100 constants: BurstGPT-like 3.73, OpenVid-like 0.096
    assert abs(T.density(*T.request_key(728, 256, 8_030_261_248, 4096, 32), A100_TF, A100_BW, 131072) / 3.73 - 1) < 0.02


def test_root_key_adds_disjoint_subtrees_and_sharing_ratio():
    # two disjoint trees: the root key is the sum of the top-level keys; a batch of identical
    # prompts shares (N-1)/N of its prompt GEMM tokens, here with d = 0
    rng = np.random.default_rng(3)
    a, b = list(rng.integers(1000, 32000, 50)), list(rng.integers(1000, 32000, 70))
    w = from_paths([a + [1], a + [2], b + [3]], p=[51, 51, 71], d=[5, 6, 7])
    v = T.build(w)
    tops = [i for i in range(v["n_nodes"]) if v["node_parent"][i] < 0]
    assert len(tops) == 2
    assert T.root_key(v) == (sum(v["cu"][i] for i in tops), sum(v["mu"][i] for i in tops))
    w2 = from_paths([a] * 4, p=[50] * 4, d=[0] * 4)
    v2 = T.build(w2)
    Pm, HL4 = 8_030_261_248, 4 * 4096 * 32
    s = T.sharing_ratio(w2, v2)
    assert s == pytest.approx(1 - (2 * Pm * 50 + HL4 * 4 * 2500) / (4 * (2 * Pm * 50 + HL4 * 2500)), rel=1e-12)


# ---------------------------------------------------------------------------
# Alg. 2 conditional node splitting (body missing -> reading #24)
# ---------------------------------------------------------------------------
def _fig_overview(prefix_len=50):
    """P:349's scenario: request #2 (low density, long output) shares a prefix with the
    compute-intensive #1 and #3; another subtree (#4, #5) sits between them in density."""
    rng = np.random.default_rng(11)
    pa = list(rng.integers(1000, 32000, prefix_len))
    pb = list(rng.integers(1000, 32000, 60))
    tail = lambda: list(rng.integers(1000, 32000, 40))    # noqa: E731
    paths = [pa + tail(), pa + tail(), pa + tail(), pb + tail(), pb + tail()]
    n = [len(x) for x in paths]
    return from_paths(paths, p=n, d=[2, 16384, 2, 300, 300])


def test_alg2_relocates_figure_outlier():
    w = _fig_overview()
    v0 = T.build(w)
    assert list(v0["req_group"]) == [0] * 5
    v = T.build(w, split_waste=50)
    # request #2 (index 1) is relocated: before, its 16K-token output dragged its
    # compute-intensive siblings' subtree below the other one; after, the siblings lead the
    # DFS order and the outlier is rightmost, so densities fall left to right
    assert list(v["req_group"]) == [0, 1, 0, 0, 0]
    assert [int(x) for x in v0["dfs_order"]] == [3, 4, 0, 2, 1]
    assert [int(x) for x in v["dfs_order"]] == [0, 2, 3, 4, 1]
    from fractions import Fraction as Fr
    tops = [i for i in range(v["n_nodes"]) if v["node_parent"][i] < 0]
    rhos = [Fr(v["cu"][i], v["mu"][i]) for i in tops]
    assert rhos == sorted(rhos, reverse=True) and len(tops) == 3
    # its 50-token shared prefix is duplicated: +50 tokens of nodes, and the batch's GEMM
    # tokens grow by exactly those 50 recomputed prompt tokens ("recomputation waste")
    assert int(v["node_len"].sum()) - int(v0["node_len"].sum()) == 50
    assert T.root_key(v)[0] - T.root_key(v0)[0] == 2 * int(w.model_params) * 50
    assert T.root_key(v)[1] == T.root_key(v0)[1]
    # every request still ends exactly once (leaf multiset unchanged)
    assert sorted(int(x) for x in v["dfs_order"]) == list(range(5))


def test_alg2_threshold_and_off():
    w = _fig_overview()
    assert list(T.build(w, split_waste=49)["req_group"]) == [0] * 5     # waste 50 > t
    v0, v1 = T.build(w), T.build(w, split_waste=0)
    assert T.dump(v0, w) == T.dump(v1, w)


def test_alg2_no_outlier_when_siblings_agree():
    # all children on the same side of rho(rt): nothing moves whatever the threshold
    rng = np.random.default_rng(12)
    pa = list(rng.integers(1000, 32000, 30))
    paths = [pa + list(rng.integers(1000, 32000, 10)) for _ in range(3)] + [list(rng.integers(1000, 32000, 40))]
    w = from_paths(paths, p=[len(x) for x in paths], d=[2, 3, 4, 20000])
    assert list(T.build(w, split_waste=10 ** 9)["req_group"]) == [0] * 4
