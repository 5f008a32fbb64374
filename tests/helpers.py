"""Random tiny workloads for tests (input generation only)."""
import numpy as np

from synth.workloads import Workload, LLAMA8B


def random_workload(seed, n_req=None, max_depth=4, max_seg=40, hq=2, hkv=1, d=64,
                    kv_dtype="f32", page_size=16, identical=True, scale_q=1.0,
                    tok_lo=1000, tok_hi=32000, max_q=None):
    """Random prefix forest: segments of 1..max_seg tokens, requests ending at
    leaves or internal nodes, occasional identical paths, prefill chunks that
    span node boundaries (q up to the whole path)."""
    rng = np.random.default_rng(seed)
    R = int(n_req if n_req is not None else rng.integers(1, 13))
    # grow a forest of segments
    segs = []          # (parent_index or -1, tokens)
    paths = []
    for r in range(R):
        if segs and rng.random() < 0.8:
            k = int(rng.integers(0, len(segs)))
            base = []
            x = k
            chain = []
            while x >= 0:
                chain.append(x)
                x = segs[x][0]
            for x in reversed(chain):
                base.extend(segs[x][1])
            if len(chain) < max_depth and rng.random() < 0.75:
                t = list(rng.integers(tok_lo, tok_hi, size=int(rng.integers(1, max_seg + 1))))
                segs.append((k, t))
                base = base + t
            elif identical and rng.random() < 0.5:
                pass                                   # identical path / ends at internal node
            else:
                cut = int(rng.integers(1, len(base) + 1))
                base = base[:cut]                      # ends mid-segment
        else:
            t = list(rng.integers(tok_lo, tok_hi, size=int(rng.integers(1, max_seg + 1))))
            segs.append((-1, t))
            base = t
        paths.append(np.array(base, dtype=np.int32))
    n = np.array([len(p) for p in paths])
    mq = n if max_q is None else np.minimum(n, max_q)
    q = np.array([int(rng.integers(1, m + 1)) if rng.random() < 0.5 else 1 for m in mq])
    p = np.array([int(x) + int(rng.integers(0, 20)) for x in n])
    dd = np.array([int(rng.integers(0, 300)) for _ in range(R)])
    tok_off = np.zeros(R + 1, dtype=np.int64)
    tok_off[1:] = np.cumsum(n)
    return Workload(name=f"rand{seed}", seed=seed, num_q_heads=hq, num_kv_heads=hkv, head_dim=d,
                    kv_dtype=kv_dtype, page_size=page_size,
                    model_params=LLAMA8B["model_params"], hidden=4096, layers=32,
                    tokens=np.concatenate(paths), tok_off=tok_off, q_len=q.astype(np.int32),
                    prompt_len=p.astype(np.int32), out_len=dd.astype(np.int32), scale_q=scale_q)


def from_paths(paths, q=None, p=None, d=None, hq=2, hkv=1, dim=64, page_size=16, seed=0,
               kv_dtype="f32"):
    paths = [np.asarray(x, dtype=np.int32) for x in paths]
    R = len(paths)
    n = np.array([len(x) for x in paths])
    tok_off = np.zeros(R + 1, dtype=np.int64)
    tok_off[1:] = np.cumsum(n)
    return Workload(name="paths", seed=seed, num_q_heads=hq, num_kv_heads=hkv, head_dim=dim,
                    kv_dtype=kv_dtype, page_size=page_size,
                    model_params=LLAMA8B["model_params"], hidden=4096, layers=32,
                    tokens=np.concatenate(paths) if R else np.zeros(0, np.int32), tok_off=tok_off,
                    q_len=np.asarray(q if q is not None else [1] * R, dtype=np.int32),
                    prompt_len=np.asarray(p if p is not None else n, dtype=np.int32),
                    out_len=np.asarray(d if d is not None else [16] * R, dtype=np.int32))


DEGENERATE = ["one_token", "single_prefill", "identical_decode", "identical_mixed_q", "nested",
              "long_decode"]


def degenerate_workload(case):
    """Edge-case batches (bf16, 8/2 heads, D=128, ps=64) shared by the plan-simulation
    and GPU parity tests."""
    rng = np.random.default_rng(77)
    tok = lambda n: rng.integers(1000, 32000, n).astype(np.int32)       # noqa: E731
    if case == "one_token":
        paths, q = [tok(1)], [1]
    elif case == "single_prefill":                  # causal prefill from position 0, ragged tail
        paths, q = [tok(700)], [700]
    elif case == "identical_decode":                # one node holding every request
        a = tok(500)
        paths, q = [a] * 20, [1] * 20
    elif case == "identical_mixed_q":
        a = tok(300)
        paths, q = [a] * 3, [300, 150, 1]
    elif case == "nested":                          # requests ending inside the tree (interior nodes)
        a, b, c = tok(400), tok(200), tok(300)
        paths = [a, np.concatenate([a, b]), np.concatenate([a, b, c]), np.concatenate([a, c])]
        q = [64, 1, 200, 7]
    elif case == "long_decode":                     # 64K-token context next to shorter siblings
        a = tok(32768)
        paths = [np.concatenate([a, tok(32768)])] + [np.concatenate([a, tok(100 + i)]) for i in range(3)]
        q = [1, 1, 3, 1]
    n = [len(x) for x in paths]
    return from_paths(paths, q=q, p=n, d=[8] * len(paths), hq=8, hkv=2, dim=128, page_size=64,
                      kv_dtype="bf16", seed=11)
