"""NEXT-2 dual-scanner batch former (PAPER §4.4): blend_schedule_build
is bit-exact with oracle/sched.py on random whole-workload trees, and the oracle is pinned
to the paper: the memory-partition worked example, the two equations,
conservation of every request's prompt and output tokens, and the memory bound."""
from fractions import Fraction

import numpy as np
import pytest

import paper_2411_16102_b200 as B
from harness.run import build_tree
from oracle import sched as OS
from oracle import tree as OT
from tests.helpers import from_paths, random_workload


def _prompt_workload(seed, n_req=30, tok_hi=32000, max_seg=40):
    """Whole-workload trees: each request's path is its full prompt (p = path length)
    and d a spread of output lengths (chatbot-like and video-like)."""
    w = random_workload(seed, n_req=n_req, tok_hi=tok_hi, max_seg=max_seg)
    rng = np.random.default_rng(seed)
    w.prompt_len = np.diff(w.tok_off).astype(np.int32)
    w.out_len = np.where(rng.random(w.n_req) < 0.3, rng.integers(200, 2000, w.n_req),
                         rng.integers(0, 40, w.n_req)).astype(np.int32)
    w.q_len[:] = 1
    return w


def test_partition_worked_example():
    # rho 3.73 and 0.096, target 1.27, M = 60 GB -> 19.3 / 40.7 GB (in 0.1 GB units: 600)
    ml = OS.partition(600, 373, 100, 96, 1000, 127, 100)
    assert ml == 193 and 600 - ml == 407


@pytest.mark.parametrize("seed", range(20))
def test_partition_satisfies_both_equations(seed):
    rng = np.random.default_rng(seed)
    cu = [int(x) for x in rng.integers(1, 10 ** 12, 3)]
    mu = [int(x) for x in rng.integers(1, 10 ** 9, 3)]
    (cl, ml), (ct, mt), (cr, mr) = sorted(zip(cu, mu), key=lambda x: -Fraction(*x))   # rho_L > rho_rt > rho_R
    M = 10 ** 6
    x = OS.partition(M, cl, ml, cr, mr, ct, mt)
    rl, rr, rt = Fraction(cl, ml), Fraction(cr, mr), Fraction(ct, mt)
    exact = M * (rt - rr) / (rl - rr)                       # M_L + M_R = M and the compute equation
    assert x == int(exact) and 0 <= x <= M
    assert abs((x * rl + (M - x) * rr) / M - rt) <= (rl - rr) / M


@pytest.mark.parametrize("seed", range(24))
@pytest.mark.parametrize("policy", [B.SCHED_DUAL, B.SCHED_DFS])
def test_schedule_matches_oracle(seed, policy):
    w = _prompt_workload(seed, tok_hi=1003 if seed % 3 == 0 else 32000)
    M = int([2000, 5000, 20000][seed % 3])
    chunk, budget = [(16, 64), (32, 10 ** 6), (512, 8192)][seed % 3]
    o = OS.schedule(w, OT.build(w), M, chunk=chunk, step_budget=budget,
                    policy="dual" if policy == B.SCHED_DUAL else "dfs")
    c = build_tree(w).schedule(M, chunk=chunk, step_budget=budget, policy=policy)
    assert c["n_steps"] == len(o["steps"])
    ents = [e for st in o["steps"] for e in st]
    assert list(c["step_off"]) == list(np.cumsum([0] + [len(st) for st in o["steps"]]))
    assert list(c["req"]) == [e[0] for e in ents]
    assert list(c["n_cached"]) == [e[1] for e in ents]
    assert list(c["q"]) == [e[2] for e in ents]
    assert list(c["order"]) == o["order"] and list(c["side"]) == o["side"]
    assert list(c["m_left"]) == o["m_left"]
    assert c["cached_prompt_tokens"] == o["cached_prompt_tokens"]
    assert c["optimal_cached_tokens"] == OS.optimal_cached_tokens(w, OT.build(w))


@pytest.mark.parametrize("seed", range(8))
def test_schedule_conserves_work_and_memory(seed):
    """Every request is admitted once; its prefill steps cover exactly its uncached prompt
    suffix (contiguous, ending at p), then exactly d decode steps at p+1..p+d; with one
    side (DFS policy) the active footprints never exceed M."""
    w = _prompt_workload(seed)
    v = OT.build(w)
    M = 3000
    o = OS.schedule(w, v, M, chunk=16, step_budget=64)
    assert sorted(o["order"]) == list(range(w.n_req))
    seen = {r: [] for r in range(w.n_req)}
    for st in o["steps"]:
        rs = [e[0] for e in st]
        assert len(rs) == len(set(rs))
        for r, n, q in st:
            seen[r].append((n, q))
    cached = 0
    for r, ev in seen.items():
        p, d = int(w.prompt_len[r]), int(w.out_len[r])
        pre = [(n, q) for n, q in ev if n <= p and q >= 1 and (n, q) != (p + 1, 1)][:len(ev) - d]
        dec = ev[len(pre):]
        assert [n for n, _ in dec] == list(range(p + 1, p + d + 1)) and all(q == 1 for _, q in dec)
        start = pre[0][0] - pre[0][1]
        for (n0, _), (n1, q1) in zip(pre, pre[1:]):
            assert n1 - q1 == n0
        assert pre[-1][0] == p
        cached += start
    assert cached == o["cached_prompt_tokens"]
    # memory (one side, fixed M: the DFS policy): the active footprints never exceed M
    # unless a single request is active
    od = OS.schedule(w, v, M, chunk=16, step_budget=64, policy="dfs")
    for st in od["steps"]:
        tot = sum(int(w.prompt_len[r]) + int(w.out_len[r]) for r, _, _ in st)
        assert tot <= M or len(st) == 1


def test_dual_scanner_blends_both_sides():
    """Two groups of opposite density under separate system prompts: the left cursor
    serves the compute-intensive group, the right the memory-intensive one, concurrently
    (P:359); the DFS order runs them one after the other."""
    rng = np.random.default_rng(4)
    sa, sb = list(rng.integers(1000, 32000, 64)), list(rng.integers(1000, 32000, 64))
    paths = [sa + list(rng.integers(1000, 32000, 30)) for _ in range(20)] + \
            [sb + list(rng.integers(1000, 32000, 30)) for _ in range(20)]
    w = from_paths(paths, p=[94] * 40, d=[2] * 20 + [3000] * 20)
    v = OT.build(w)
    o = OS.schedule(w, v, 2000, chunk=64, step_budget=4096)
    assert set(o["side"][:20]) == {0}
    # the right cursor starts on the memory-intensive group; once the left cursor has
    # drained its group the cursors meet and both sides draw from the last unit
    assert o["side"][o["order"][[r >= 20 for r in o["order"]].index(True)]] == 1
    first = o["steps"][0]
    assert {r < 20 for r, _, _ in first} == {True, False}          # both sides in the first batch
    od = OS.schedule(w, v, 2000, chunk=64, step_budget=4096, policy="dfs")
    assert {r < 20 for r, _, _ in od["steps"][0]} == {True}


def test_c4_whole_workload_sharing_and_blending():
    """The C4 grid as a whole offline workload (40,000 requests, full prompts) on one B200's
    KV capacity (1.2M tokens): the dual scanner keeps > 97 % of the optimal prefix sharing
    (">99 %") and, by blending both ends of the sorted tree, needs fewer
    steps than the DFS order for the same tokens."""
    from synth import workloads as W
    w = W.c4_grid(whole=True)
    t = build_tree(w)
    dual = t.schedule(1_200_000, policy=B.SCHED_DUAL)
    dfs = t.schedule(1_200_000, policy=B.SCHED_DFS)
    assert dual["cached_prompt_tokens"] >= 0.97 * dual["optimal_cached_tokens"]
    assert dfs["cached_prompt_tokens"] >= 0.97 * dfs["optimal_cached_tokens"]
    assert sorted(dual["order"]) == list(range(w.n_req))
    assert dual["n_steps"] < dfs["n_steps"]
    # both sides are in use from the first step (the memory partition of P:362-368)
    first = dual["req"][dual["step_off"][0]:dual["step_off"][1]]
    assert set(dual["side"][first].tolist()) == {0, 1}
