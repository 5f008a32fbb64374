"""GPU parity: libblend (through the C ABI) vs the fp64 oracle, element by element.

Tolerances (BASELINE north_star, reading #22): bf16 KV -> max |O - O*| <= 2e-2
and ||O - O*||_F / ||O*||_F <= 1e-2, |lse - lse*| <= 1e-3; fp32 debug path ->
1e-5 for all three.  Generator bit-exactness and paging/order invariances are
checked bitwise."""
import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

import paper_2411_16102_b200 as B  # noqa: E402
from harness.run import device_batch, page_slot_hashes, query_rows  # noqa: E402
from oracle import attention as A  # noqa: E402
from synth import values as V  # noqa: E402
from synth import workloads as W  # noqa: E402
from tests.helpers import random_workload  # noqa: E402

TOL = {"bf16": (2e-2, 1e-2, 1e-3), "f32": (1e-5, 1e-5, 1e-5)}
PATHS = [B.PATH_AUTO, B.PATH_GENERIC, B.PATH_NO_TCGEN05]


def _cmp(w, db, requests=None, tol=None):
    atol, rtol, ltol = tol or TOL[w.kv_dtype]
    ref = A.attention_workload(w, requests)
    out = db.out.float().cpu().numpy()
    lse = db.lse.cpu().numpy()
    qo = np.concatenate([[0], np.cumsum(w.q_len)])
    num = den = 0.0
    worst = 0.0
    for r, (O, L) in ref.items():
        o = out[qo[r]:qo[r + 1]]
        l = lse[qo[r]:qo[r + 1]]
        assert np.all(np.isfinite(o)) and np.all(np.isfinite(l)), f"request {r}: non-finite"
        worst = max(worst, float(np.max(np.abs(o - O))))
        assert np.max(np.abs(l - L)) <= ltol, (r, float(np.max(np.abs(l - L))))
        num += float(np.sum((o - O) ** 2))
        den += float(np.sum(O ** 2))
    rel = np.sqrt(num / max(den, 1e-300))
    assert worst <= atol and rel <= rtol, f"max abs {worst:.3e} (atol {atol}), rel {rel:.3e} (rtol {rtol}), {_where(w, db, ref)}"

    return worst


def _where(w, db, ref):
    """Locate the worst rows (request, query, head) to make a failure diagnosable."""
    out = db.out.float().cpu().numpy()
    qo = np.concatenate([[0], np.cumsum(w.q_len)])
    worst = []
    for r, (O, L) in ref.items():
        err = np.abs(out[qo[r]:qo[r + 1]] - O).max(axis=-1)        # [q, Hq]
        t, h = np.unravel_index(np.argmax(err), err.shape)
        worst.append((float(err[t, h]), r, int(t), int(h)))
    worst.sort(reverse=True)
    bad_heads = sorted({h for e, _, _, h in worst if e > 1e-2})
    return f"worst (err, req, t, head) = {worst[:4]}, heads over 1e-2: {bad_heads[:16]}"


@pytest.fixture(scope="module", autouse=True)
def _cuda():
    if not torch.cuda.is_available():
        pytest.skip("no GPU")
    B.lib()


def test_fill_matches_generator():
    w = W.c1_tiny("d", "f32")
    db = device_batch(w)
    pid, pcnt, phash = page_slot_hashes(w, db.view)
    kc = db.k_cache.cpu().numpy()
    vc = db.v_cache.cpu().numpy()
    for i in range(len(pid)):
        h = phash[i * w.page_size: i * w.page_size + pcnt[i]]
        K = V.kv_values(h, w.seed, 0, w.num_kv_heads, w.head_dim)
        Vv = V.kv_values(h, w.seed, 1, w.num_kv_heads, w.head_dim)
        assert np.array_equal(kc[pid[i], :, :pcnt[i]].transpose(1, 0, 2), K)
        assert np.array_equal(vc[pid[i], :, :pcnt[i]].transpose(1, 0, 2), Vv)
        assert np.all(kc[pid[i], :, pcnt[i]:] == 0)
    gid, tt = query_rows(w)
    q = db.q.cpu().numpy()
    for i in range(len(gid)):
        assert np.array_equal(q[i], V.q_values(int(gid[i]), np.array([tt[i]]), w.seed,
                                               w.num_q_heads, w.head_dim)[0])


def test_fill_bf16_matches_generator():
    w = W.c2_mmlu_decode(n_req=8)
    w.scale_q = 8.0
    db = device_batch(w)
    gid, tt = query_rows(w)
    q = db.q.float().cpu().numpy()
    for i in range(len(gid)):
        assert np.array_equal(q[i], V.q_values(int(gid[i]), np.array([tt[i]]), w.seed,
                                               w.num_q_heads, w.head_dim, 8.0)[0])


@pytest.mark.parametrize("mode", ["a", "b", "c", "d"])
def test_c1_fp32(mode):
    w = W.c1_tiny(mode, "f32")
    for kw in (dict(), dict(force_class=1), dict(rows_min=1, min_sep_len=0), dict(split_tokens=16)):
        db = device_batch(w, tree_kw=kw)
        db.run()
        torch.cuda.synchronize()
        _cmp(w, db)


@pytest.mark.parametrize("mode", ["a", "b", "c", "d"])
@pytest.mark.parametrize("path", PATHS)
def test_c1_bf16(mode, path):
    w = W.c1_tiny(mode, "bf16")
    for kw in (dict(), dict(force_class=1), dict(force_class=2), dict(rows_min=1, min_sep_len=0),
               dict(split_tokens=16)):
        db = device_batch(w, tree_kw=kw)
        db.run(path=path)
        torch.cuda.synchronize()
        _cmp(w, db)


@pytest.mark.parametrize("path", PATHS)
@pytest.mark.parametrize("scale_q", [1.0, 8.0])
def test_c2_full(path, scale_q):
    w = W.c2_mmlu_decode()
    w.scale_q = scale_q
    db = device_batch(w)
    assert db.info["n_dense_units"] > 0 and db.info["n_stream_units"] > 0
    db.run(path=path)
    torch.cuda.synchronize()
    _cmp(w, db)


@pytest.mark.parametrize("seed", range(8))
def test_random_trees_bf16(seed):
    hq, hkv = [(8, 2), (32, 8), (16, 1), (4, 4)][seed % 4]
    w = random_workload(seed, hq=hq, hkv=hkv, d=128 if seed % 2 else 64, kv_dtype="bf16",
                        page_size=[16, 32, 64, 128][seed % 4], max_seg=300, n_req=int(8 + seed * 5))
    for kw in (dict(), dict(force_class=1, min_sep_len=0), dict(rows_min=16, min_sep_len=0)):
        db = device_batch(w, tree_kw=kw)
        for path in PATHS:
            db.out.zero_()
            db.run(path=path)
            torch.cuda.synchronize()
            _cmp(w, db)


def test_page_permutation_and_classes_invariance():
    w = W.c2_mmlu_decode(n_req=64)
    db = device_batch(w)
    db.run()
    base = db.out.clone()
    perm = np.random.default_rng(0).permutation(5000).astype(np.int32)
    db2 = device_batch(w, tree_kw=dict(free_pages=perm))
    db2.run()
    torch.cuda.synchronize()
    assert torch.equal(base, db2.out), "page-id permutation changed the output"
    # literal cascade vs all-folded: same attention within tolerance
    db3 = device_batch(w, tree_kw=dict(force_class=1))
    db3.run()
    db4 = device_batch(w, tree_kw=dict(force_class=2))
    db4.run()
    torch.cuda.synchronize()
    assert (db3.out.float() - db4.out.float()).abs().max().item() < 2e-2


@pytest.mark.parametrize("name", ["c3", "c4", "c5"])
def test_large_configs_sampled(name):
    """Full-size C3 / C5 in the bench's launch configuration, checked on a
    stratified request sample (BIG/SMALL, shortest/longest contexts)."""
    w = W.by_name(name)
    db = device_batch(w)
    db.run()
    torch.cuda.synchronize()
    n = np.diff(w.tok_off)
    big = np.nonzero(w.q_len * (w.num_q_heads // w.num_kv_heads) >= 128)[0]
    small = np.nonzero(w.q_len * (w.num_q_heads // w.num_kv_heads) < 128)[0]
    pick = set(big[:3].tolist()) | set(small[np.argsort(n[small])[:3]].tolist()) \
        | set(small[np.argsort(n[small])[-3:]].tolist())
    rng = np.random.default_rng(0)
    pick |= set(rng.choice(w.n_req, size=6, replace=False).tolist())
    _cmp(w, db, sorted(pick))


def test_request_order_invariance():
    """Permuting the caller's request order leaves every request's rows bitwise equal
    (each row's arithmetic does not depend on which other rows share its tile)."""
    from harness.run import subset
    w = W.c2_mmlu_decode(n_req=48)
    db = device_batch(w)
    db.run()
    perm = np.random.default_rng(3).permutation(w.n_req)
    w2 = subset(w, perm)                      # global ids travel with the requests
    db2 = device_batch(w2)
    db2.run()
    torch.cuda.synchronize()
    a, b = db.out.cpu(), db2.out.cpu()
    for i, r in enumerate(perm):
        assert torch.equal(a[r], b[i]), r


def test_abi_errors():
    w = W.c1_tiny("a", "bf16")
    db = device_batch(w, tree_kw=dict(force_class=1, min_sep_len=0))
    with pytest.raises(B.BlendError) as e:
        B.attention(db.q, db.k_cache, db.v_cache, db.plan, db.out, db.lse, db.ws[:16],
                    n_cache_pages=db.n_cache_pages)
    assert e.value.status == B.ENOSPC
    with pytest.raises(B.BlendError) as e:
        B.attention(db.q, db.k_cache, db.v_cache, db.plan, db.out, db.lse, db.ws,
                    n_cache_pages=db.n_cache_pages, path=7)
    assert e.value.status == B.EINVAL
    # a plan page id beyond the cache allocation -> EINVAL (not a silent zero-filled read)
    assert db.plan.max_page == int(db.view["page_table"].max())
    with pytest.raises(B.BlendError) as e:
        B.attention(db.q, db.k_cache, db.v_cache, db.plan, db.out, db.lse, db.ws,
                    n_cache_pages=db.plan.max_page)
    assert e.value.status == B.EINVAL
    # q / out of another dtype than the plan's kv_dtype -> EINVAL
    with pytest.raises(B.BlendError) as e:
        B.attention(db.q.float(), db.k_cache, db.v_cache, db.plan, db.out.float(), db.lse, db.ws,
                    n_cache_pages=db.n_cache_pages)
    assert e.value.status == B.EINVAL


@pytest.mark.parametrize("flags", [0, 1])
def test_c2_overlap_bitwise(flags):
    """The PDL overlap of the two passes and the serialised launch give the same bits."""
    w = W.c2_mmlu_decode()
    db = device_batch(w)
    db.run(flags=flags)
    torch.cuda.synchronize()
    _cmp(w, db)
    first = db.out.clone()
    db.run(flags=1 - flags)
    torch.cuda.synchronize()
    assert torch.equal(first, db.out)


@pytest.mark.parametrize("hq,hkv,d,ps", [(6, 3, 128, 64), (12, 4, 64, 32), (8, 1, 128, 128), (10, 2, 128, 16)])
def test_group_sizes_bf16(hq, hkv, d, ps):
    """GQA group sizes 2, 3, 8, 5: g = 3 and 5 do not divide a 128-row tile (dense units
    gather Q rows with cp.async, tiles split tokens), g = 2 / 8 use the TMA Q boxes;
    page sizes 16..128 exercise the multi-entry 64-key blocks."""
    w = random_workload(100 + hq, hq=hq, hkv=hkv, d=d, kv_dtype="bf16", page_size=ps, max_seg=300,
                        n_req=24)
    for kw in (dict(), dict(force_class=1, min_sep_len=0), dict(rows_min=8, min_sep_len=0)):
        db = device_batch(w, tree_kw=kw)
        db.run()
        torch.cuda.synchronize()
        _cmp(w, db)


@pytest.mark.parametrize("name,G", [("c2", 2), ("c2", 4), ("c5", 8), ("c2x2", 2)])
def test_sharded_equals_single_gpu(name, G):
    """§8(e) invariant "G-GPU == 1-GPU" on one device, through the bench's own DP code
    (harness/dp.py): ONE global batch (c2x2: two independent C2 copies) is sharded by
    blend_shard into G subtree shards, each shard planned, filled and run on its own, and
    the rows re-assembled in global request order by row_index (what gather_rows does after
    the all-gather) equal the unsharded run within the bf16 tolerance (different plans,
    so not bitwise) and match the oracle on sampled requests."""
    from harness.dp import row_index, shard_batch
    if name == "c2x2":
        gw = W.replicate(lambda seed: W.c2_mmlu_decode(n_req=48, seed=seed), 2, 2)
    else:
        gw = W.by_name(name)
    dbg = device_batch(gw)
    dbg.run()
    torch.cuda.synchronize()
    full_o, full_l = dbg.out.float().cpu(), dbg.lse.cpu()
    del dbg
    got_o = torch.full_like(full_o, float("nan"))
    got_l = torch.full_like(full_l, float("nan"))
    for g in range(G):
        ws, req_shard, _ = shard_batch(gw, G, g)
        assert ws.n_req > 0
        if name == "c5" and G == 8:   # P:246 / SURVEY c-5: subtree snapping -> 2 whole documents per GPU
            docs = {int(ws.path(r)[256]) for r in range(ws.n_req)}
            assert len(docs) == 2 and ws.n_req == 128
        db = device_batch(ws)
        db.run()
        torch.cuda.synchronize()
        ix = torch.from_numpy(row_index(gw, req_shard, G)[g])
        got_o[ix] = db.out.float().cpu()
        got_l[ix] = db.lse.cpu()
        _cmp(ws, db, requests=list(range(0, ws.n_req, max(1, ws.n_req // 4))))
        del db
    assert not torch.isnan(got_l).any(), "every row in exactly one shard"
    assert (got_o - full_o).abs().max().item() <= 2e-2
    assert (got_l - full_l).abs().max().item() <= 1e-3


@pytest.mark.parametrize("n", [2, 4, 8])
def test_tp_slices_concat_to_full(n):
    """NEXT-4 head parallelism on the full C5 batch (70B shapes, 64/8 heads): rank k
    of n runs kv heads [8k/n, 8(k+1)/n) with global head indices in the synthetic values;
    the n slices concatenated along the head axis equal the full-head run bitwise (same
    split-KV plan: split sizes pinned) and match the oracle on sampled requests."""
    from dataclasses import replace
    from harness.dp import tp_heads
    gw = W.c5_70b_32k()
    kw = dict(split_tokens=4096, dense_split=2)
    full = device_batch(gw, tree_kw=kw)
    full.run()
    torch.cuda.synchronize()
    fo, fl = full.out.cpu(), full.lse.cpu()
    del full
    outs, lses = [], []
    for k in range(n):
        hq, hkv, h0, kvh0 = tp_heads(gw, n, k)
        w = replace(gw, num_q_heads=hq, num_kv_heads=hkv, head0=h0, kv_head0=kvh0)
        db = device_batch(w, tree_kw=kw)
        db.run()
        torch.cuda.synchronize()
        outs.append(db.out.cpu())
        lses.append(db.lse.cpu())
        if k == n - 1:
            _cmp(w, db, requests=[0, 63, 500, 1023])      # the slice against the oracle's heads
        del db
    assert torch.equal(torch.cat(outs, dim=1), fo)
    assert torch.equal(torch.cat(lses, dim=1), fl)


@pytest.mark.parametrize("seed", range(8, 16))
def test_random_trees_bf16_long(seed):
    """Longer nodes (up to 400 tokens per segment): multi-block dense
    units, split-KV streaming, partial tiles and causal diagonals at scale."""
    hq, hkv = [(8, 1), (8, 2), (32, 8), (16, 4)][seed % 4]
    w = random_workload(seed, hq=hq, hkv=hkv, d=128 if seed % 3 else 64, kv_dtype="bf16",
                        page_size=[64, 16, 32, 128][seed % 4], max_seg=400, n_req=int(12 + seed))
    for kw in (dict(), dict(force_class=1, min_sep_len=0), dict(split_tokens=128)):
        db = device_batch(w, tree_kw=kw)
        db.run()
        torch.cuda.synchronize()
        _cmp(w, db)


@pytest.mark.parametrize("seed", range(4))
def test_random_trees_fp32(seed):
    """fp32 debug path (generic FMA executor + merge kernel) on random forests, 1e-5."""
    hq, hkv = [(2, 1), (4, 2), (8, 1), (4, 4)][seed]
    w = random_workload(200 + seed, hq=hq, hkv=hkv, d=64 if seed % 2 else 128, kv_dtype="f32",
                        page_size=[16, 32, 64, 128][seed], max_seg=120, n_req=10 + 3 * seed)
    for kw in (dict(), dict(force_class=1, min_sep_len=0), dict(split_tokens=32)):
        db = device_batch(w, tree_kw=kw)
        db.run()
        torch.cuda.synchronize()
        _cmp(w, db)


@pytest.mark.parametrize("case", ["one_token", "single_prefill", "identical_decode",
                                  "identical_mixed_q", "nested", "long_decode"])
@pytest.mark.parametrize("path", PATHS)
@pytest.mark.parametrize("kw", [dict(), dict(force_class=1, min_sep_len=0, dense_split=3),
                                dict(force_class=2, split_tokens=64)])
def test_degenerate_shapes(case, path, kw):
    """Edge cases of the method: a one-token batch, a full causal prefill, identical paths
    (one node, no private suffix), requests that end at interior nodes, a 64K context."""
    from tests.helpers import degenerate_workload
    w = degenerate_workload(case)
    db = device_batch(w, tree_kw=kw)
    db.run(path=path)
    torch.cuda.synchronize()
    _cmp(w, db)


@pytest.mark.parametrize("seed", range(3))
def test_alg2_split_trees(seed):
    """NEXT-3: trees rebuilt by Alg. 2 (relocated subtrees with duplicated prefix pages) give
    the same attention (P:346-351 changes descriptors, not the attention definition)."""
    w = random_workload(600 + seed, hq=8, hkv=2, d=128, kv_dtype="bf16", page_size=64, max_seg=300,
                        n_req=24, tok_hi=1003 if seed == 0 else 32000)
    for t_w in (64, 10 ** 6):
        db = device_batch(w, tree_kw=dict(split_waste=t_w))
        db.run()
        torch.cuda.synchronize()
        _cmp(w, db)


def test_scheduled_steps_parity():
    """NEXT-2: blended batches formed by the dual scanner from a small whole workload
    (full prompts, mixed output lengths) are ordinary attention steps: sampled steps
    (prefill chunks next to decodes, prefixes reused from other requests) match the oracle."""
    from synth.workloads import step_workload
    from harness.run import build_tree
    rng = np.random.default_rng(9)
    sysp = list(rng.integers(1000, 32000, 200))
    paths = [sysp + list(rng.integers(1000, 32000, int(rng.integers(50, 700)))) for _ in range(40)]
    from tests.helpers import from_paths
    w = from_paths(paths, p=[len(x) for x in paths], d=[2] * 20 + [400] * 20, hq=32, hkv=8, dim=128,
                   page_size=64, kv_dtype="bf16")
    sched = build_tree(w).schedule(6000, chunk=256, step_budget=1024)
    so = sched["step_off"]
    S = sched["n_steps"]
    for s in sorted({0, 1, 3, S // 3, S // 2, S - 1}):
        a, b = int(so[s]), int(so[s + 1])
        sw = step_workload(w, sched["req"][a:b], sched["n_cached"][a:b], sched["q"][a:b])
        db = device_batch(sw)
        db.run()
        torch.cuda.synchronize()
        _cmp(sw, db)
