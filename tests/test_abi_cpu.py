"""C-ABI checks that need no GPU: the library loads and exports the header's
symbols; descriptors, rejections, shards and dumps are bit-exact with the
oracle; the device plan, interpreted on the CPU, reproduces the oracle."""
import os
import re

import numpy as np
import pytest

import paper_2411_16102_b200 as B
from harness.run import build_tree
from oracle import attention as A
from oracle import shard as OS
from oracle import tree as OT
from synth import workloads as W
from tests.helpers import DEGENERATE, degenerate_workload, random_workload
from tests.plan_sim import simulate

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
KEYS = ["n_nodes", "node_parent", "node_start", "node_len", "node_page_off", "node_class",
        "node_key_cu", "node_key_mu", "node_first_req", "node_nreq", "page_table", "req_path_off",
        "req_path_nodes", "req_q_off", "req_class", "req_dfs_rank", "req_global_id", "req_group"]


def test_exports_every_header_symbol():
    hdr = open(os.path.join(ROOT, "include", "blend.h")).read()
    names = set(re.findall(r"^\s*(?:const\s+)?[a-z_0-9]+\**\s+\**(blend_[a-z_0-9]+)\s*\(", hdr, re.M))
    assert len(names) >= 15, names
    L = B.lib()
    for n in sorted(names):
        assert hasattr(L, n), n
    assert L.blend_abi_version() == 2


def _same(v_c, v_o):
    for k in KEYS:
        a, b = np.asarray(v_c[k]), np.asarray(v_o[k])
        assert a.shape == b.shape and np.array_equal(a.astype(np.int64) if a.dtype != np.uint64 else a,
                                                     b.astype(np.int64) if b.dtype != np.uint64 else b), k


KW = [dict(), dict(min_sep_len=0), dict(force_class=1), dict(force_class=2, min_sep_len=0),
      dict(rows_min=1, min_sep_len=0), dict(rows_min=4, min_sep_len=8)]


@pytest.mark.parametrize("seed", range(30))
def test_descriptors_random(seed):
    hq, hkv = [(1, 1), (2, 1), (4, 2), (8, 1)][seed % 4]
    w = random_workload(seed, hq=hq, hkv=hkv, page_size=[16, 32, 64, 128][seed % 4],
                        tok_hi=1004 if seed % 5 == 0 else 32000)
    kw = KW[seed % len(KW)]
    free = np.random.default_rng(seed).permutation(20000).astype(np.int32) if seed % 2 else None
    v_o = OT.build(w, free_pages=free, **{"rows_min": 128, "min_sep_len": 128, **kw})
    t = build_tree(w, free_pages=free, **{"rows_min": 128, "min_sep_len": 128, **kw})
    _same(t.view(), v_o)
    assert t.dump() == OT.dump(v_o, w)


@pytest.mark.parametrize("seed", range(16))
def test_descriptors_alg2_split(seed):
    """Alg. 2 conditional node splitting (split_waste = t): bit-exact with the oracle,
    and the plan of the split tree still computes exact attention (CPU plan interpreter)."""
    w = random_workload(500 + seed, hq=4, hkv=2, tok_hi=1004 if seed % 3 == 0 else 32000, max_seg=30,
                        n_req=int(10 + seed))
    t_w = [4, 20, 60, 10 ** 6][seed % 4]
    v_o = OT.build(w, split_waste=t_w)
    t = build_tree(w, split_waste=t_w)
    _same(t.view(), v_o)
    assert t.dump() == OT.dump(v_o, w)
    if seed % 4 == 1:
        out, lse, written, _ = simulate(w, t)
        ref = A.attention_workload(w)
        qo = np.concatenate([[0], np.cumsum(w.q_len)])
        for r, (O, L) in ref.items():
            assert np.max(np.abs(out[qo[r]:qo[r + 1]] - O)) < 1e-10


def test_alg2_relocates_somewhere():
    moved = 0
    for seed in range(16):
        w = random_workload(500 + seed, hq=4, hkv=2, tok_hi=1004 if seed % 3 == 0 else 32000, max_seg=30,
                            n_req=int(10 + seed))
        moved += int((OT.build(w, split_waste=10 ** 6)["req_group"] > 0).sum())
    assert moved > 0


@pytest.mark.parametrize("name", ["c1a", "c1b", "c1c", "c1d", "c2", "c3", "c5"])
def test_descriptors_configs(name):
    w = W.by_name(name)
    v_o = OT.build(w)
    t = build_tree(w)
    _same(t.view(), v_o)


def test_big_keys_exact():
    # 70B constants and 16K outputs push CU past 2^64: the 128-bit keys must still agree
    w = W.c5_70b_32k(n_docs=3, per_doc=4, doc_len=512)
    w.out_len[:] = 500_000_000 + np.arange(w.n_req)
    w.prompt_len[:] = 1_000_000_000 - 7 * np.arange(w.n_req)
    v_o = OT.build(w)
    t = build_tree(w)
    _same(t.view(), v_o)
    assert max(v_o["cu"]) > 2**80 and max(v_o["mu"]) > 2**62


@pytest.mark.parametrize("bad", ["q0", "qbig", "empty", "noreq", "negtok", "heads", "dim", "ps", "nospc", "dup"])
def test_rejections_match(bad):
    from tests.helpers import from_paths
    w = from_paths([[1, 2, 3], [1, 2, 4]])
    fp = None
    if bad == "q0":
        w.q_len[0] = 0
    elif bad == "qbig":
        w.q_len[0] = 4
    elif bad == "empty":
        w = from_paths([[1, 2, 3], []])
    elif bad == "noreq":
        w = from_paths([])
    elif bad == "negtok":
        w.tokens[1] = -5
    elif bad == "heads":
        w.num_q_heads, w.num_kv_heads = 3, 2
    elif bad == "dim":
        w.head_dim = 96
    elif bad == "ps":
        w.page_size = 24
    elif bad == "nospc":
        fp = np.array([0, 1], np.int32)
    elif bad == "dup":
        fp = np.array([0, 1, 1, 3], np.int32)
    with pytest.raises(OT.BlendError) as eo:
        OT.build(w, free_pages=fp)
    with pytest.raises(B.BlendError) as ec:
        build_tree(w, free_pages=fp)
    assert eo.value.status == ec.value.status


@pytest.mark.parametrize("seed", range(12))
def test_shard_matches_oracle(seed):
    w = random_workload(seed, n_req=int(np.random.default_rng(seed).integers(1, 30)))
    t = build_tree(w)
    v = OT.build(w)
    for G in (1, 2, 3, 4, 8):
        rs_o = OS.shard_assign(w, v, G)
        rs_c, shards = t.shard(G)
        assert np.array_equal(rs_o, rs_c), G
        subs = OS.shard_workloads(w, rs_o, G)
        for g in range(G):
            if subs[g].n_req == 0:
                assert shards[g] is None
                continue
            _same(shards[g].view(), OT.build(subs[g]))


@pytest.mark.parametrize("name,G", [("c2", 8), ("c5", 8), ("c3", 4)])
def test_shard_configs(name, G):
    w = W.by_name(name)
    t = build_tree(w)
    rs_c, _ = t.shard(G)
    assert np.array_equal(rs_c, OS.shard_assign(w, OT.build(w), G))


def _check_sim(w, **kw):
    t = build_tree(w, **kw)
    out, lse, written, _ = simulate(w, t)
    assert np.all(written == 1), "every (token, head) written exactly once"
    ref = A.attention_workload(w)
    qo = np.concatenate([[0], np.cumsum(w.q_len)])
    for r in range(w.n_req):
        O, L = ref[r]
        assert np.max(np.abs(out[qo[r]:qo[r + 1]] - O)) < 1e-10
        assert np.max(np.abs(lse[qo[r]:qo[r + 1]] - L)) < 1e-10
    return t


@pytest.mark.parametrize("seed", range(16))
def test_plan_simulation_random(seed):
    hq, hkv = [(1, 1), (2, 1), (4, 2), (8, 1)][seed % 4]
    w = random_workload(seed, hq=hq, hkv=hkv, page_size=[16, 32, 64, 128][(seed // 4) % 4],
                        max_seg=90)
    kw = dict(KW[seed % len(KW)])
    kw.setdefault("rows_min", 128)
    kw.setdefault("min_sep_len", 128)
    if seed % 3 == 0:
        kw["split_tokens"] = 64
    _check_sim(w, **kw)


@pytest.mark.parametrize("mode", ["a", "b", "c", "d"])
@pytest.mark.parametrize("kw", [dict(), dict(force_class=1), dict(rows_min=1, min_sep_len=0),
                                dict(split_tokens=16)])
def test_plan_simulation_c1(mode, kw):
    _check_sim(W.c1_tiny(mode), **kw)


def test_plan_simulation_c2_small():
    w = W.c2_mmlu_decode(n_req=24)
    t = _check_sim(w, rows_min=64)
    info = t.plan_info()
    assert info["n_dense_units"] > 0 and info["n_stream_units"] > 0


@pytest.mark.parametrize("seed", range(4))
def test_plan_simulation_mixed_sep_rows(seed):
    """SEPARATE items mixing prefill rows of several requests (unsorted positions)."""
    hq, hkv = [(8, 2), (32, 8), (16, 1), (4, 4)][seed % 4]
    w = random_workload(seed, hq=hq, hkv=hkv, d=128 if seed % 2 else 64, kv_dtype="bf16",
                        page_size=[16, 32, 64, 128][seed % 4], max_seg=200, n_req=int(6 + seed * 2),
                        max_q=64)
    for kw in (dict(), dict(force_class=1, min_sep_len=0), dict(rows_min=16, min_sep_len=0)):
        _check_sim(w, **kw)


@pytest.mark.parametrize("hq,hkv,d,ps", [(6, 3, 128, 64), (12, 4, 64, 32), (8, 1, 128, 128), (10, 2, 128, 16)])
def test_plan_simulation_group_sizes(hq, hkv, d, ps):
    """Planner + plan image for GQA groups 2, 3, 8, 5 (tiles that split tokens when
    g does not divide 128) reproduce the oracle in fp64 simulation."""
    w = random_workload(100 + hq, hq=hq, hkv=hkv, d=d, kv_dtype="f32", page_size=ps, max_seg=300, n_req=24)
    for kw in (dict(), dict(force_class=1, min_sep_len=0), dict(rows_min=8, min_sep_len=0)):
        _check_sim(w, **kw)


def test_dense_grid_cap():
    """The planner caps the dense grid only when the dense pass alone would fill the GPU
    and both passes are large (C4, C5 shapes); a small dense pass (C2) or a
    streaming-dominated batch (C3) keeps one CTA per SM."""
    import ctypes as C
    L = B.lib()
    f = L.blend_internal_dense_ctas
    f.restype, f.argtypes = C.c_int32, [C.c_void_p]
    caps = {n: f(build_tree(W.by_name(n), num_sms=148).handle) for n in ("c2", "c3", "c4", "c5")}
    assert caps["c2"] == 0 and caps["c3"] == 0
    for n in ("c4", "c5"):
        assert int(0.4 * 148) <= caps[n] < 148, caps


def test_plan_simulation_stream_tail_split():
    """Streaming tail balance: with 40 decodes x 8 kv heads = 320 streaming units on
    4 x 13 = 52 rings the last round would be 8 units, so the planner splits the
    shortest items in two; the plan still reproduces the oracle and every split token
    gets one more source."""
    w = W.c2_mmlu_decode(n_req=40)
    t0 = build_tree(w, num_sms=16)           # 320 % 64 == 0: no split
    t1 = _check_sim(w, num_sms=13)           # 320 % 52 == 8: split
    i0, i1 = t0.plan_info(), t1.plan_info()
    assert i1["n_stream_units"] > i0["n_stream_units"]
    assert i1["n_partial_rows"] > i0["n_partial_rows"]


@pytest.mark.parametrize("case", DEGENERATE)
@pytest.mark.parametrize("kw", [dict(), dict(force_class=1, min_sep_len=0, dense_split=3),
                                dict(force_class=2, split_tokens=64)])
def test_plan_simulation_degenerate(case, kw):
    """The plan of each edge-case batch computes the oracle's attention in fp64."""
    _check_sim(degenerate_workload(case), **kw)
