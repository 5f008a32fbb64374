"""CPU interpreter of libblend's device plan (test infrastructure).

Reads the plan image the C++ planner produced (internal symbol
blend_internal_plan_image), executes every work unit in fp64 numpy exactly as
the kernels are specified to (keys of the unit's page entries, per-row causal
mask, partial (o, lse) or direct write per the partmap), merges the partials
in the plan's order, and returns (out, lse) — so the host planner is checked
against the oracle without a GPU."""
import ctypes as C

import numpy as np

import paper_2411_16102_b200 as B
from harness.run import page_slot_hashes, query_rows
from oracle import attention as A
from synth import values as V

SEC = ["tok_pos", "item_tok_off", "item_tokens", "entries", "dunits", "sunits", "partmap",
       "merge_tok", "merge_off", "stream_rows", "dense_qtok", "dunits_ks", "dense_ks_qtok"]


def plan_image(tree):
    L = B.lib()
    f = L.blend_internal_plan_image
    f.restype = C.c_int
    f.argtypes = [C.c_void_p, C.POINTER(C.c_void_p), C.POINTER(C.c_size_t),
                  C.POINTER(C.POINTER(C.c_int64)), C.POINTER(C.POINTER(C.c_int64))]
    data, nbytes = C.c_void_p(), C.c_size_t()
    off, cnt = C.POINTER(C.c_int64)(), C.POINTER(C.c_int64)()
    assert f(tree.handle, C.byref(data), C.byref(nbytes), C.byref(off), C.byref(cnt)) == 0
    blob = np.ctypeslib.as_array(C.cast(data, C.POINTER(C.c_uint8)), (nbytes.value,)).copy() \
        if nbytes.value else np.zeros(0, np.uint8)
    secs = {}
    width = {"entries": 4, "dunits": 8, "sunits": 8, "stream_rows": 4, "dunits_ks": 8}
    for i, name in enumerate(SEC):
        o, n = int(off[i]), int(cnt[i])
        k = width.get(name, 1)
        secs[name] = blob[o:o + 4 * n * k].view(np.int32).reshape(n, k) if k > 1 else \
            blob[o:o + 4 * n].view(np.int32)
    return secs


STREAM_ROWS = 16


def check_stream_rows(P, g, Hq):
    """The planner's per-row descriptors of streaming units restate (item row ->
    token, head, position, partmap target) exactly."""
    sr = P["stream_rows"]
    assert len(sr) == STREAM_ROWS * len(P["sunits"])
    for ui, u in enumerate(P["sunits"]):
        item, kvh, rb, nr, eb, ee, pmb, tb = (int(x) for x in u)
        for r in range(STREAM_ROWS):
            qrow, pos, tgt, head = (int(x) for x in sr[ui * STREAM_ROWS + r])
            if r >= nr:
                assert qrow == -1 and tgt == -2
                continue
            tl, j = (rb + r) // g, (rb + r) % g
            tok = int(P["item_tokens"][tb + tl])
            assert (qrow, pos, tgt, head) == (tok * Hq + kvh * g + j, int(P["tok_pos"][tok]),
                                              int(P["partmap"][pmb + tl]), kvh * g + j)


def check_dense_qtok(P, g, ps):
    """A dense unit marked for TMA Q loading (first token t0 >= 0) covers whole tokens
    t0, t0+1, ... of q; every unit with consecutive whole tokens is marked when its
    128-row tiles hold whole tokens.  Key-split units (dense_ks.cu) are exactly the bf16
    units of <= 128 rows and >= 2 64-key blocks."""
    epb = 64 // min(ps, 64)
    for name, qname, ks in (("dunits", "dense_qtok", False), ("dunits_ks", "dense_ks_qtok", True)):
        for u in P[name]:
            nr, ne = int(u[3]), int(u[5]) - int(u[4])
            assert (nr <= 128 and (ne + epb - 1) // epb >= 2) == ks or (not ks and len(P["dunits_ks"]) == 0), \
                (name, nr, ne)
    _check_qtok(P["dense_qtok"], P["dunits"], P, g)
    _check_qtok(P["dense_ks_qtok"], P["dunits_ks"], P, g)


def _check_qtok(qt, dunits, P, g):
    assert len(qt) == len(dunits)
    for ui, u in enumerate(dunits):
        item, kvh, rb, nr, eb, ee, pmb, tb = (int(x) for x in u)
        toks = [int(P["item_tokens"][tb + tl]) for tl in range(rb // g, (rb + nr - 1) // g + 1)]
        consec = rb % g == 0 and toks == list(range(toks[0], toks[0] + len(toks)))
        if 256 % g == 0 and 128 % g == 0:
            assert int(qt[ui]) == (toks[0] if consec else -1), (ui, int(qt[ui]), toks[:4])
        else:
            assert int(qt[ui]) == -1


def simulate(w, tree):
    view = tree.view()
    P = plan_image(tree)
    g = w.num_q_heads // w.num_kv_heads
    D, Hq, Hkv, ps = w.head_dim, w.num_q_heads, w.num_kv_heads, w.page_size
    pid, pcnt, phash = page_slot_hashes(w, view)
    page_index = {int(p): i for i, p in enumerate(pid)}
    gid, tt = query_rows(w)
    T = len(gid)
    Q = np.zeros((T, Hq, D))
    for i in range(T):
        Q[i] = V.q_values(int(gid[i]), np.array([tt[i]]), w.seed, Hq, D, w.scale_q, w.head0)[0]
    nprow = tree.plan_info()["n_partial_rows"]
    part_o = np.full((nprow, Hq, D), np.nan)
    part_l = np.full((nprow, Hq), np.nan)
    out = np.full((T, Hq, D), np.nan)
    lse = np.full((T, Hq), np.nan)
    written = np.zeros((T, Hq), dtype=np.int64)
    check_stream_rows(P, g, Hq)
    check_dense_qtok(P, g, ps)
    for kind, units in (("dense", P["dunits"]), ("dense", P["dunits_ks"]), ("stream", P["sunits"])):
        for u in units:
            item, kvh, rb, nr, eb, ee, pmb, tb = (int(x) for x in u)
            kpos, K, Vv = [], [], []
            for e in range(eb, ee):
                page, roff, pos0, cnt = (int(x) for x in P["entries"][e])
                pi = page_index[page]
                h = phash[pi * ps + roff: pi * ps + roff + cnt]
                K.append(V.kv_values(h, w.seed, 0, Hkv, D, w.kv_head0)[:, kvh])
                Vv.append(V.kv_values(h, w.seed, 1, Hkv, D, w.kv_head0)[:, kvh])
                kpos.extend(range(pos0, pos0 + cnt))
            K = np.concatenate(K)[:, None, :]
            Vv = np.concatenate(Vv)[:, None, :]
            for r in range(nr):
                ir = rb + r
                tl, j = ir // g, ir % g
                tok = int(P["item_tokens"][tb + tl])
                head = kvh * g + j
                pos = int(P["tok_pos"][tok])
                o, l = A.partial(K, Vv, Q[tok:tok + 1, head:head + 1], [pos], kpos)
                tgt = int(P["partmap"][pmb + tl])
                if tgt == -2:
                    continue
                if tgt == -1:
                    out[tok, head], lse[tok, head] = o[0, 0], l[0, 0]
                    written[tok, head] += 1
                else:
                    assert np.isnan(part_l[tgt, head]), "partial row written twice"
                    part_o[tgt, head], part_l[tgt, head] = o[0, 0], l[0, 0]
    mo = P["merge_off"]
    assert int(mo[-1]) == nprow
    for m, tok in enumerate(P["merge_tok"]):
        rows = list(range(int(mo[m]), int(mo[m + 1])))   # list m = partial rows mo[m] .. mo[m+1]-1
        assert len(rows) >= 2
        assert not np.isnan(part_l[rows]).any(), "merge reads an unwritten partial"
        for h in range(Hq):
            parts = [(part_o[r, h][None, None], part_l[r, h][None, None]) for r in rows]
            O, L = A.lse_merge(parts)
            out[tok, h], lse[tok, h] = O[0, 0], L[0, 0]
        written[tok] += 1
    return out, lse, written, P
