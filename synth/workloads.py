"""Seeded synthetic workloads shaped like the paper's traces.

INPUT GENERATION ONLY — no method arithmetic lives here.  Each recipe returns a
`Workload`: per-request cached token paths (CSR), the number of this step's
query tokens q_r (the last q_r tokens of the path), the prompt length p_r and
(estimated) output length d_r used only for density ordering, and the model /
cache shape.

Token ids are U[1000, 32000); every trace gets its own system
prompt.  Lognormals are parameterised by their MEAN and sigma.
"""
from __future__ import annotations

import json
import os
from dataclasses import dataclass, field, replace
from typing import List, Optional

import numpy as np

LLAMA8B = dict(model_params=8_030_261_248, hidden=4096, layers=32,
               num_q_heads=32, num_kv_heads=8, head_dim=128)
LLAMA70B = dict(model_params=70_553_706_496, hidden=8192, layers=80,
                num_q_heads=64, num_kv_heads=8, head_dim=128)

TOK_LO, TOK_HI = 1000, 32000


@dataclass
class Workload:
    name: str
    seed: int
    num_q_heads: int
    num_kv_heads: int
    head_dim: int
    kv_dtype: str               # "bf16" | "f32"
    page_size: int
    model_params: int
    hidden: int
    layers: int
    tokens: np.ndarray          # int32[sum n_r]
    tok_off: np.ndarray         # int64[R+1]
    q_len: np.ndarray           # int32[R]
    prompt_len: np.ndarray      # int32[R]
    out_len: np.ndarray         # int32[R]
    scale_q: float = 1.0
    free_pages: Optional[np.ndarray] = None   # int32 physical page ids, None = 0,1,2,...
    global_id: Optional[np.ndarray] = None    # int64[R] global request index (Q generator)
    head0: int = 0                            # global index of q head 0 (head-parallel slices)
    kv_head0: int = 0                         # global index of kv head 0
    meta: dict = field(default_factory=dict)

    @property
    def n_req(self) -> int:
        return int(self.q_len.shape[0])

    def path(self, r: int) -> np.ndarray:
        return self.tokens[self.tok_off[r]:self.tok_off[r + 1]]

    def path_len(self) -> np.ndarray:
        return np.diff(self.tok_off)

    def gid(self, r: int) -> int:
        return int(self.global_id[r]) if self.global_id is not None else r

    @property
    def sum_q(self) -> int:
        return int(self.q_len.sum())


def _toks(rng, n):
    return rng.integers(TOK_LO, TOK_HI, size=n, dtype=np.int64).astype(np.int32)


def _lognormal_mean(rng, mean, sigma, size, lo, hi):
    mu = np.log(mean) - 0.5 * sigma * sigma
    x = np.rint(rng.lognormal(mu, sigma, size=size)).astype(np.int64)
    return np.clip(x, lo, hi)


def _pack(name, seed, paths: List[np.ndarray], q, p, d, dims, kv_dtype, page_size, **kw) -> Workload:
    tok_off = np.zeros(len(paths) + 1, dtype=np.int64)
    tok_off[1:] = np.cumsum([len(x) for x in paths])
    tokens = np.concatenate(paths).astype(np.int32) if paths else np.zeros(0, np.int32)
    return Workload(name=name, seed=seed, kv_dtype=kv_dtype, page_size=page_size,
                    tokens=tokens, tok_off=tok_off,
                    q_len=np.asarray(q, dtype=np.int32), prompt_len=np.asarray(p, dtype=np.int32),
                    out_len=np.asarray(d, dtype=np.int32), **dims, **kw)


def c1_tiny(mode: str = "a", kv_dtype: str = "f32", seed: int = 1) -> Workload:
    """configs[0]: 8 requests share a 64-token system prompt; suffixes 16..48 tokens;
    Hq=2, Hkv=1, D=64; ps=16; physical pages permuted by the seed.
    modes: a decode q=1 | b suffix prefill q=s_r | c (b) + pseudo-request #8 = the
    prompt with q=64 | d two groups of 4 under 16-token group prefixes, mixed q."""
    rng = np.random.default_rng(seed)
    sys_p = _toks(rng, 64)
    s = rng.integers(16, 49, size=8)
    suffix = [_toks(rng, int(x)) for x in s]
    gp = [_toks(rng, 16), _toks(rng, 16)]
    paths, q, p, d = [], [], [], []
    for r in range(8):
        if mode == "d":
            path = np.concatenate([sys_p, gp[r // 4], suffix[r]])
            qq = 1 if r % 2 == 0 else int(s[r])
            pp = 80 + int(s[r])
        else:
            path = np.concatenate([sys_p, suffix[r]])
            qq = 1 if mode == "a" else int(s[r])
            pp = 64 + int(s[r])
        paths.append(path); q.append(qq); p.append(pp); d.append(16)
    if mode == "c":
        paths.append(sys_p.copy()); q.append(64); p.append(64); d.append(16)
    dims = dict(model_params=LLAMA8B["model_params"], hidden=4096, layers=32,
                num_q_heads=2, num_kv_heads=1, head_dim=64)
    free = rng.permutation(4096).astype(np.int32)
    return _pack(f"c1{mode}_{kv_dtype}", seed, paths, q, p, d, dims, kv_dtype, 16, free_pages=free)


def c2_mmlu_decode(seed: int = 2, n_req: int = 256) -> Workload:
    """configs[1]: Llama-3.1-8B shapes, decode batch 256 over one shared 1024-token
    MMLU-like prefix (64 system + 960 five-shot); private = question U{79..119}
    + 1 generated token; q=1; p = 1024+u, d = 2 (MMLU answers)."""
    rng = np.random.default_rng(seed)
    shared = _toks(rng, 1024)
    u = rng.integers(79, 120, size=n_req)
    paths = [np.concatenate([shared, _toks(rng, int(x) + 1)]) for x in u]
    return _pack("c2_mmlu_decode", seed, paths, np.ones(n_req), 1024 + u, np.full(n_req, 2),
                 dict(LLAMA8B), "bf16", 64)


def c3_burst_openvid(seed: int = 3, n_prefill: int = 64, n_video: int = 960) -> Workload:
    """configs[2]: 64 BurstGPT chunked prefills (system 128, chunk start c0 in
    {0,512,1024}, q=512) + 960 OpenVid decodes at ~16K context (system 128,
    caption U{60..140}, generated U{12000..20000}, q=1, d = 80 frames x 256)."""
    rng = np.random.default_rng(seed)
    sys_b, sys_v = _toks(rng, 128), _toks(rng, 128)
    paths, q, p, d = [], [], [], []
    c0 = rng.choice([0, 512, 1024], size=n_prefill)
    dl = _lognormal_mean(rng, 256, 0.7, n_prefill, 1, 4096)
    extra = rng.integers(0, 512, size=n_prefill)
    for i in range(n_prefill):
        paths.append(np.concatenate([sys_b, _toks(rng, int(c0[i]) + 512)]))
        q.append(512); p.append(128 + int(c0[i]) + 512 + int(extra[i])); d.append(int(dl[i]))
    cap = rng.integers(60, 141, size=n_video)
    gen = rng.integers(12000, 20001, size=n_video)
    for i in range(n_video):
        paths.append(np.concatenate([sys_v, _toks(rng, int(cap[i]) + int(gen[i]))]))
        q.append(1); p.append(128 + int(cap[i])); d.append(20480)
    return _pack("c3_burst_openvid", seed, paths, q, p, d, dict(LLAMA8B), "bf16", 64)


def c5_70b_32k(seed: int = 5, n_docs: int = 16, per_doc: int = 64, doc_len: int = 30720) -> Workload:
    """configs[4]: Llama-3.1-70B shapes; system 256 -> 16 documents x 30720 tokens
    -> 64 requests each with private U{1536..2560}; q=1; context ~33K."""
    rng = np.random.default_rng(seed)
    sys_p = _toks(rng, 256)
    paths, q, p, d = [], [], [], []
    for _ in range(n_docs):
        doc = _toks(rng, doc_len)
        priv = rng.integers(1536, 2561, size=per_doc)
        for x in priv:
            paths.append(np.concatenate([sys_p, doc, _toks(rng, int(x))]))
            q.append(1); p.append(256 + doc_len + 128); d.append(4096)
    return _pack("c5_70b_32k", seed, paths, q, p, d, dict(LLAMA70B), "bf16", 64)


C4_COUNTS_PATH = os.path.join(os.path.dirname(os.path.abspath(__file__)), "c4_counts.json")
C4_T = (0.8, 1.0, 1.2, 1.4)


def c4_counts(t: float):
    """(BurstGPT, OpenVid, MMLU) request counts of the C4 grid at density t: the table
    written by scripts/solve_c4_counts.py (solved on the realised samples with the
    oracle's density keys)."""
    with open(C4_COUNTS_PATH) as f:
        table = json.load(f)
    e = table["t"][f"{t:.1f}"]
    return tuple(int(x) for x in e["counts"])


def c4_grid(seed: int = 4, t: float = 1.0, counts=None, chunk: int = 512, n_total: int = 40000,
            whole: bool = False) -> Workload:
    """configs[3]: the paper's A.1 grid recipe with synthetic lengths —
    40,000 requests mixing BurstGPT-like (prompt LN(600, 0.7) in [16, 4096], output
    LN(256, 0.7) in [1, 4096]), OpenVid-like (caption LN(100, 0.4) in [16, 512],
    frames LN(64, 0.3) in [8, 256], d = 256 tokens per frame, mean 16384) and
    MMLU-like requests (57 subjects with a 5-shot prefix U{400..1000}, question
    LN(100, 0.4) in [20, 400], d = 2); 3-level tree: trace system prompt (128)
    -> MMLU subject -> request.  Counts (Burst, OpenVid, MMLU) for compute density t and
    sharing s = 0.5 come from c4_counts(t) unless given.
    Each class draws from its own random stream, so the first n requests of a class do
    not depend on the other classes' counts (the count solve is monotone).
    Snapshot: every request sits at a uniformly random step of its lifetime
    (ceil(p_private / 512) prefill chunks, then d decodes); shared prefixes cached.
    whole=True: the whole offline workload instead (NEXT-2): each path is the request's
    full prompt (p = path length), for the dual-scanner batch former."""
    nb, nv, nm = c4_counts(t) if counts is None else counts
    rs = np.random.default_rng([seed, 0])
    sys_b, sys_v, sys_m = _toks(rs, 128), _toks(rs, 128), _toks(rs, 128)
    subj = [_toks(rs, int(rs.integers(400, 1001))) for _ in range(57)]
    paths, q, p, d = [], [], [], []

    def snapshot(rng, shared, priv_len, dd):
        if whole:
            return np.concatenate([shared, _toks(rng, priv_len)]), 1
        n_chunks = -(-priv_len // chunk)
        k = int(rng.integers(0, n_chunks + dd))
        if k < n_chunks:
            cached = min((k + 1) * chunk, priv_len)
            qq = cached - k * chunk
            priv = _toks(rng, cached)
        else:
            priv = _toks(rng, priv_len + (k - n_chunks) + 1)
            qq = 1
        return np.concatenate([shared, priv]), qq

    rb = np.random.default_rng([seed, 1])
    for _ in range(nb):
        pb = int(_lognormal_mean(rb, 600, 0.7, 1, 16, 4096)[0])
        db = int(_lognormal_mean(rb, 256, 0.7, 1, 1, 4096)[0])
        path, qq = snapshot(rb, sys_b, pb, db)
        paths.append(path); q.append(qq); p.append(128 + pb); d.append(db)
    rv = np.random.default_rng([seed, 2])
    # d = 256 tokens per frame; E[frames] = 64 -> mean d = 16384
    for _ in range(nv):
        cap = int(_lognormal_mean(rv, 100, 0.4, 1, 16, 512)[0])
        frames = int(_lognormal_mean(rv, 64, 0.3, 1, 8, 256)[0])
        dv = 256 * frames
        path, qq = snapshot(rv, sys_v, cap, dv)
        paths.append(path); q.append(qq); p.append(128 + cap); d.append(dv)
    rm = np.random.default_rng([seed, 3])
    for _ in range(nm):
        qm = int(_lognormal_mean(rm, 100, 0.4, 1, 20, 400)[0])
        sm = int(rm.integers(0, 57))
        shared = np.concatenate([sys_m, subj[sm]])
        path, qq = snapshot(rm, shared, qm, 2)
        paths.append(path); q.append(qq); p.append(len(shared) + qm); d.append(2)
    order = np.random.default_rng([seed, 9]).permutation(len(paths))   # arrival order is not tree order
    w = _pack(f"c4_{'whole' if whole else 'grid'}_t{t:.1f}_s0.5", seed, [paths[i] for i in order], np.asarray(q)[order],
              np.asarray(p)[order], np.asarray(d)[order], dict(LLAMA8B), "bf16", 64)
    w.meta.update(counts=(nb, nv, nm), t=t)
    return w


def generated_tokens(w: Workload, r: int, n: int) -> np.ndarray:
    """Synthetic output tokens 0..n-1 of request r (whole-workload runs): a counter hash of
    (seed, global request id, index), ids in [TOK_LO, TOK_HI)."""
    from synth import values as V
    ctr = (np.uint64(w.gid(r)) << np.uint64(24)) + np.arange(n, dtype=np.uint64)
    z = V.mix(np.uint64(w.seed ^ 0x6A09E667F3BCC909) ^ V.mix(ctr))
    return (TOK_LO + (z % np.uint64(TOK_HI - TOK_LO)).astype(np.int64)).astype(np.int32)


def step_workload(w: Workload, req, n_cached, q, name: str = "step") -> Workload:
    """The blended batch of one scheduled step: request req[i] with cached path length
    n_cached[i] (its prompt prefix, then its generated tokens) and q[i] query tokens."""
    paths = []
    for r, n in zip(req, n_cached):
        r, n = int(r), int(n)
        pr = w.path(r)
        paths.append(pr[:n] if n <= len(pr) else np.concatenate([pr, generated_tokens(w, r, n - len(pr))]))
    tok_off = np.zeros(len(paths) + 1, dtype=np.int64)
    tok_off[1:] = np.cumsum([len(x) for x in paths])
    gid = np.asarray([w.gid(int(r)) for r in req], dtype=np.int64)
    return Workload(name=name, seed=w.seed, num_q_heads=w.num_q_heads, num_kv_heads=w.num_kv_heads,
                    head_dim=w.head_dim, kv_dtype=w.kv_dtype, page_size=w.page_size,
                    model_params=w.model_params, hidden=w.hidden, layers=w.layers,
                    tokens=np.concatenate(paths).astype(np.int32), tok_off=tok_off,
                    q_len=np.asarray(q, dtype=np.int32), prompt_len=w.prompt_len[np.asarray(req)],
                    out_len=w.out_len[np.asarray(req)], scale_q=w.scale_q, global_id=gid)


def concat(workloads: List[Workload], name: str) -> Workload:
    """Union of independent workloads (weak-scaling global batch).  Global ids are
    positions in the union; the union's value seed (K/V/Q generator) is the first
    part's.  Parts made with different recipe seeds have distinct system prompts,
    so their prefix trees are disjoint."""
    w0 = workloads[0]
    paths, q, p, d = [], [], [], []
    for w in workloads:
        for r in range(w.n_req):
            paths.append(w.path(r))
        q.append(w.q_len); p.append(w.prompt_len); d.append(w.out_len)
    dims = dict(model_params=w0.model_params, hidden=w0.hidden, layers=w0.layers,
                num_q_heads=w0.num_q_heads, num_kv_heads=w0.num_kv_heads, head_dim=w0.head_dim)
    return _pack(name, w0.seed, paths, np.concatenate(q), np.concatenate(p), np.concatenate(d),
                 dims, w0.kv_dtype, w0.page_size, scale_q=w0.scale_q)


def replicate(make, n: int, base_seed: int) -> Workload:
    """n independent copies of a recipe (seeds base_seed, base_seed+1000, ...)."""
    parts = [make(seed=base_seed + 1000 * i) for i in range(n)]
    return concat(parts, f"{parts[0].name}_x{n}")


def by_name(name: str) -> Workload:
    table = {
        "c1a": lambda: c1_tiny("a"), "c1b": lambda: c1_tiny("b"),
        "c1c": lambda: c1_tiny("c"), "c1d": lambda: c1_tiny("d"),
        "c1a_bf16": lambda: c1_tiny("a", "bf16"), "c1b_bf16": lambda: c1_tiny("b", "bf16"),
        "c1c_bf16": lambda: c1_tiny("c", "bf16"), "c1d_bf16": lambda: c1_tiny("d", "bf16"),
        "c2": c2_mmlu_decode, "c3": c3_burst_openvid, "c4": c4_grid, "c5": c5_70b_32k,
    }
    for t in C4_T:
        table[f"c4_t{t:.1f}"] = (lambda t_=t: c4_grid(t=t_))
    return table[name]()


def with_scale_q(w: Workload, scale_q: float) -> Workload:
    return replace(w, scale_q=scale_q)
