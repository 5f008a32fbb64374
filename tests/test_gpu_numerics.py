"""GPU parity under peaked score distributions, planted needles and poisoned page tails.

Uniform Q (scale 1) gives near-flat softmax rows, which never exercise the kernels'
rescaling paths.  These tests drive them on purpose and prove it with the library's
diagnostic path counters (blend_internal_set_stats, csrc/common.cuh STAT_*):

  * dense pass: the max-first ("slow") softmax path after a unit's first block and the
    lazy O rescale in TMEM (running max grows by > 2^8, dense.cu);
  * streaming pass: online-softmax rescales of live rows;
  * both passes: the zeroing of V rows past an entry's count, with those slots holding
    NaN (blend.h: slots past a node's end may hold anything).

Every result is compared with the fp64 oracle at the north-star tolerance (reading #22).
"""
import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

import paper_2411_16102_b200 as B  # noqa: E402
from harness.run import device_batch, page_slot_hashes  # noqa: E402
from oracle import attention as A  # noqa: E402
from synth import values as V  # noqa: E402
from synth import workloads as W  # noqa: E402
from tests.helpers import degenerate_workload, random_workload  # noqa: E402
from tests.test_gpu_parity import PATHS, TOL, _cmp  # noqa: E402


@pytest.fixture(scope="module", autouse=True)
def _cuda():
    if not torch.cuda.is_available():
        pytest.skip("no GPU")
    B.lib()


def _stats_run(db, **kw):
    buf = torch.zeros(8, dtype=torch.int64, device="cuda")
    B.set_stats(buf)
    try:
        db.run(**kw)
        torch.cuda.synchronize()
    finally:
        B.set_stats(None)
    return dict(zip(B.STAT_NAMES, buf.cpu().tolist()))


def _poison_tails(w, db):
    """Write NaN into every K/V slot past a node's end (the tail of its last page)."""
    pid, pcnt, _ = page_slot_hashes(w, db.view)
    nan = float("nan")
    for p, c in zip(pid.tolist(), pcnt.tolist()):
        if c < w.page_size:
            db.k_cache[p, :, c:, :] = nan
            db.v_cache[p, :, c:, :] = nan
    torch.cuda.synchronize()


def _plant_needles(w, db, picks, scale=8.0):
    """Q row (request r, query t, head h) := scale * K[key position, kvh]: a planted needle
    (SURVEY §8(c-5)).  Returns {r: Q[q_r, Hq, D]} (fp64) for the oracle."""
    g = w.num_q_heads // w.num_kv_heads
    qo = np.concatenate([[0], np.cumsum(w.q_len)])
    qs = {}
    for r, t, h, kpos in picks:
        if r not in qs:
            qs[r] = V.q_values(w.gid(r), np.arange(int(w.q_len[r])), w.seed, w.num_q_heads, w.head_dim,
                               w.scale_q)
        K, _ = V.path_kv(w.path(r), w.seed, w.num_kv_heads, w.head_dim)
        qs[r][t, h] = scale * K[kpos, h // g]
        dt = torch.bfloat16 if w.kv_dtype == "bf16" else torch.float32
        db.q[qo[r] + t, h] = torch.from_numpy(qs[r][t, h]).to(dt).cuda()
    torch.cuda.synchronize()
    return qs


def _cmp_needles(w, db, qs):
    atol, rtol, ltol = TOL[w.kv_dtype]
    out = db.out.float().cpu().numpy()
    lse = db.lse.cpu().numpy()
    qo = np.concatenate([[0], np.cumsum(w.q_len)])
    for r, Q in qs.items():
        K, Vv = V.path_kv(w.path(r), w.seed, w.num_kv_heads, w.head_dim)
        O, L = A.attention_request(K, Vv, Q, int(w.q_len[r]))
        o, l = out[qo[r]:qo[r + 1]], lse[qo[r]:qo[r + 1]]
        assert np.all(np.isfinite(o))
        err = float(np.max(np.abs(o - O)))
        rel = float(np.linalg.norm(o - O) / np.linalg.norm(O))
        assert err <= atol and rel <= rtol, (r, err, rel)
        assert float(np.max(np.abs(l - L))) <= ltol * max(1.0, float(np.max(np.abs(L)))), r


def _needle_picks(w, rng, n_pick, late_frac=0.6, want_big=None):
    """(r, t, h, key position) with the key in the last (1 - late_frac) of the visible range
    of query t, so the needle lands in a late 64-key block."""
    g = w.num_q_heads // w.num_kv_heads
    n = np.diff(w.tok_off)
    cand = [r for r in range(w.n_req) if n[r] >= 200]
    if want_big is not None:
        cand = [r for r in cand if (int(w.q_len[r]) * g >= 128) == want_big]
    picks = []
    for r in rng.choice(cand, size=min(n_pick, len(cand)), replace=False):
        r = int(r)
        q = int(w.q_len[r])
        for t in sorted({q - 1, int(rng.integers(0, q))}):
            pos = int(n[r]) - q + t
            kpos = int(rng.integers(int(late_frac * pos), pos + 1))
            picks.append((r, t, int(rng.integers(0, w.num_q_heads)), kpos))
    return picks


@pytest.mark.parametrize("seed", range(6))
def test_random_trees_peaked(seed):
    """Peaked Q (scale 8: bf16-exact k/16 values, score std ~ 2.7) on random forests with
    long nodes, the three kernel paths and three plan shapes; the counters show that the
    dense late max-first path, the dense lazy O rescale (a jump of > 2^8 over the running
    max) and the streaming rescale all fired (B200 run: 110..2100 lazy rescales per seed)."""
    hq, hkv = [(8, 2), (32, 8), (16, 4)][seed % 3]
    w = random_workload(300 + seed, hq=hq, hkv=hkv, d=128 if seed % 2 == 0 else 64, kv_dtype="bf16",
                        page_size=[64, 16, 32][seed % 3], max_seg=400, n_req=int(14 + 2 * seed), scale_q=8.0)
    tot = dict.fromkeys(B.STAT_NAMES, 0)
    for kw in (dict(), dict(force_class=1, min_sep_len=0), dict(rows_min=16, min_sep_len=0)):
        db = device_batch(w, tree_kw=kw)
        for path in PATHS:
            db.out.zero_()
            st = _stats_run(db, path=path)
            _cmp(w, db)
            if path == B.PATH_AUTO:
                for k in tot:
                    tot[k] += st[k]
    assert tot["dense_blocks"] > 0 and tot["stream_stages"] > 0, tot
    assert tot["dense_slow_late"] > 0 and tot["dense_rescale"] > 0, tot
    assert tot["stream_rescale"] > 0 and tot["tail_zeroed"] > 0, tot
    print("path counters", tot)


@pytest.mark.parametrize("case", ["single_prefill", "identical_decode", "nested", "long_decode"])
def test_degenerate_peaked(case):
    w = degenerate_workload(case)
    w.scale_q = 8.0
    for kw in (dict(), dict(force_class=1, min_sep_len=0, dense_split=3), dict(force_class=2, split_tokens=64)):
        db = device_batch(w, tree_kw=kw)
        for path in PATHS:
            db.out.zero_()
            db.run(path=path)
            torch.cuda.synchronize()
            _cmp(w, db)


@pytest.mark.parametrize("mode", ["a", "b", "c", "d"])
def test_c1_peaked(mode):
    w = W.c1_tiny(mode, "bf16")
    w.scale_q = 8.0
    for kw in (dict(), dict(force_class=1), dict(rows_min=1, min_sep_len=0), dict(split_tokens=16)):
        db = device_batch(w, tree_kw=kw)
        for path in PATHS:
            db.run(path=path)
            torch.cuda.synchronize()
            _cmp(w, db)


def _long_separate_workload(seed):
    """64 decodes under one 2048-token shared node (SEPARATE, 32 dense blocks) plus 4
    BIG prefill chunks of 384 tokens over 1500-token private paths."""
    rng = np.random.default_rng(seed)
    shared = rng.integers(1000, 32000, 2048).astype(np.int32)
    paths, q = [], []
    for i in range(64):
        paths.append(np.concatenate([shared, rng.integers(1000, 32000, int(rng.integers(50, 300)))]))
        q.append(1)
    for i in range(4):
        paths.append(rng.integers(1000, 32000, 1500).astype(np.int32))
        q.append(384)
    from tests.helpers import from_paths
    n = [len(x) for x in paths]
    return from_paths(paths, q=q, p=n, d=[8] * len(paths), hq=32, hkv=8, dim=128, page_size=64,
                      kv_dtype="bf16", seed=seed)


def test_needles_fire_dense_lazy_rescale():
    """Planted needles (Q row = 8 x a late key) in a long SEPARATE node's rows and in long
    BIG prefills: the needle block beats the running max by >> 2^8, so the dense kernel
    must rescale O in TMEM; O ~ V_needle, any skipped rescale would be off by 2^40."""
    w = _long_separate_workload(21)
    rng = np.random.default_rng(5)
    db = device_batch(w)
    assert db.info["n_dense_units"] > 0
    picks = _needle_picks(w, rng, 6, want_big=False) + _needle_picks(w, rng, 3, want_big=True)
    qs = _plant_needles(w, db, picks)
    st = _stats_run(db)
    _cmp_needles(w, db, qs)
    assert st["dense_rescale"] > 0 and st["dense_slow_late"] > 0, st
    for path in (B.PATH_GENERIC, B.PATH_NO_TCGEN05):
        db.out.zero_()
        db.run(path=path)
        torch.cuda.synchronize()
        _cmp_needles(w, db, qs)


def test_needles_c2_streaming():
    """C2 (SURVEY d-4: needles on C1/C2): needles in the private suffixes (streaming pass)
    and in the shared 1K prefix (dense pass)."""
    w = W.c2_mmlu_decode(n_req=96)
    db = device_batch(w)
    rng = np.random.default_rng(2)
    picks = []
    for r in rng.choice(w.n_req, size=12, replace=False):
        n = len(w.path(int(r)))
        kpos = int(rng.integers(1030, n)) if len(picks) % 2 == 0 else int(rng.integers(600, 1024))
        picks.append((int(r), 0, int(rng.integers(0, 32)), kpos))
    qs = _plant_needles(w, db, picks)
    st = _stats_run(db)
    _cmp_needles(w, db, qs)
    assert st["stream_rescale"] > 0 and st["dense_rescale"] > 0, st


@pytest.mark.parametrize("seed", range(4))
def test_nan_page_tails(seed):
    """Slots past a node's end hold NaN in K and V: every path stays finite and within
    tolerance (the kernels zero those V rows; masked scores discard the K rows)."""
    hq, hkv = [(8, 2), (32, 8), (4, 1), (16, 4)][seed]
    w = random_workload(400 + seed, hq=hq, hkv=hkv, d=128 if seed % 2 == 0 else 64, kv_dtype="bf16",
                        page_size=[64, 16, 32, 128][seed], max_seg=300, n_req=int(16 + seed))
    for kw in (dict(), dict(force_class=1, min_sep_len=0, dense_split=2), dict(rows_min=16, min_sep_len=0)):
        db = device_batch(w, tree_kw=kw)
        _poison_tails(w, db)
        for path in PATHS:
            db.out.zero_()
            st = _stats_run(db, path=path)
            _cmp(w, db)
            if path == B.PATH_AUTO:
                assert st["tail_zeroed"] > 0, st


def test_nan_page_tails_fp32():
    w = random_workload(450, hq=4, hkv=2, d=64, kv_dtype="f32", page_size=32, max_seg=100, n_req=10)
    db = device_batch(w, tree_kw=dict(force_class=1, min_sep_len=0))
    _poison_tails(w, db)
    db.run()
    torch.cuda.synchronize()
    _cmp(w, db)
