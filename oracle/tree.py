"""Descriptor oracle — independent Python re-implementation of the rules that
`blend_tree_build` must reproduce bit-exactly.

TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).

Rules, each with the passage it follows:
 1. Trie ("each leaf node ... represents an actual request while each
    internal node is a segment of the prefix shared by all its descendants";
    P:6 "construct a prefix tree following a Trie Tree"): nodes are maximal
    runs of path positions over which the set A(pi) of requests having prefix
    pi is constant, so a node boundary falls at every divergence and at every
    request end (SPEC S:154-155 examples).  Built here by plain radix insertion.
 2. Density key (P:87-96 cost model, P:309-320 density of a node = over all
    requests in its subtree, P:315 rho(R) = (1-s) T_comp / T_mem):
      G_S  = sum_{N in closure(S)} clamp(maxP_S(N) - start(N), 0, len(N))
             + sum_{r in S} max(0, p_r - n_r) + sum_{r in S} d_r
      CU_S = 2 P_model G_S + 4 H L sum_{r in S} p_r^2
      MU_S = sum_{r in S} (p_r d_r + d_r (d_r + 1) / 2)
    (hardware constants and H_kv*L*4 cancel in comparisons: readings #8-#10).
 3. Sort (Alg 1, body missing -> reading #11): children of every
    node and the top-level forest ordered by rho descending:
      a before b iff MU_a = 0 < MU_b, or (MU_a, MU_b > 0 and CU_a MU_b > CU_b MU_a);
    equal keys -> smaller minimum request id in the subtree.
 4. Numbering: node id = preorder index of the sorted forest; request DFS order
    = at each node the requests ending there (ascending id), then the children.
 5. Pages: nodes in id order take ceil(len/ps) consecutive free-list entries.
 6. Classes (§8(a-4); ">= 128 shared tokens"; P:14 multiples of 128):
    request BIG iff q_r g >= rows_min; node SEPARATE iff |A(N)| >= 2 and
    g * sum_{r in A(N), SMALL} q_r >= rows_min and len(N) >= min_sep_len.
    force_class 1: every shared node SEPARATE (for all its requests);
    force_class 2: no node SEPARATE.
 7. Rejections: same inputs and status codes as the C-ABI (BlendError.status).
"""
from __future__ import annotations

import functools
from dataclasses import dataclass, field
from typing import Dict, List, Optional

import numpy as np

OK, EINVAL, EMALFORMED, ENOSPC, ECUDA, ENOMEM, EUNSUPPORTED = 0, -1, -2, -3, -4, -5, -6


class BlendError(Exception):
    def __init__(self, status: int, msg: str):
        super().__init__(msg)
        self.status = status


@dataclass
class _Node:
    start: int
    length: int
    ref: int                          # a request whose path spells this node's tokens
    parent: Optional["_Node"] = None
    children: Dict[int, "_Node"] = field(default_factory=dict)
    ends: List[int] = field(default_factory=list)


def _validate(w, rows_min, min_sep_len, force_class, n_free):
    hq, hkv, d, ps = w.num_q_heads, w.num_kv_heads, w.head_dim, w.page_size
    if hq <= 0 or hkv <= 0 or hq % hkv != 0:
        raise BlendError(EINVAL, "num_q_heads must be a positive multiple of num_kv_heads")
    if d not in (64, 128):
        raise BlendError(EUNSUPPORTED, "head_dim must be 64 or 128")
    if ps < 16 or ps > 128 or (ps & (ps - 1)) != 0:
        raise BlendError(EINVAL, "page_size must be a power of two in [16,128]")
    if w.kv_dtype not in ("bf16", "f32"):
        raise BlendError(EINVAL, "kv_dtype")
    if rows_min < 1 or min_sep_len < 0 or force_class not in (0, 1, 2):
        raise BlendError(EINVAL, "rows_min/min_sep_len/force_class")
    if w.n_req < 1:
        raise BlendError(EINVAL, "n_req must be >= 1")
    n = np.diff(w.tok_off)
    for r in range(w.n_req):
        if n[r] < 1:
            raise BlendError(EMALFORMED, f"request {r}: empty path")
        if w.q_len[r] < 1 or w.q_len[r] > n[r]:
            raise BlendError(EMALFORMED, f"request {r}: q_len out of range")
        if w.prompt_len[r] < 0 or w.out_len[r] < 0:
            raise BlendError(EMALFORMED, f"request {r}: negative prompt/out length")
    if w.tokens.size and int(w.tokens.min()) < 0:
        raise BlendError(EMALFORMED, "negative token id")


def _build_trie(w, group=None):
    """Radix insertion.  group[r] (Alg. 2 relocation group, 0 = none) separates requests
    at the root: relocated requests never share a node with other groups."""
    root = _Node(0, 0, -1)
    for r in range(w.n_req):
        P = w.path(r)
        n = P.shape[0]
        node, pos = root, 0
        while True:
            tok = int(P[pos])
            key = (int(group[r]) if group is not None else 0, tok) if node is root else tok
            child = node.children.get(key)
            if child is None:
                leaf = _Node(pos, n - pos, r, parent=node)
                leaf.ends.append(r)
                node.children[key] = leaf
                break
            seg = w.path(child.ref)[child.start:child.start + child.length]
            L = min(child.length, n - pos)
            neq = np.nonzero(seg[:L] != P[pos:pos + L])[0]
            k = int(neq[0]) if neq.size else L
            if k < child.length:                       # split child at k
                upper = _Node(child.start, k, child.ref, parent=node)
                node.children[key] = upper
                child.start += k
                child.length -= k
                child.parent = upper
                upper.children[int(seg[k])] = child
                child = upper
            node, pos = child, pos + k
            if pos == n:
                node.ends.append(r)
                break
    return root


def _all_nodes(root):
    out, stack = [], list(root.children.values())
    while stack:
        x = stack.pop()
        out.append(x)
        stack.extend(x.children.values())
    return out


def relocation_groups(w, view, split_waste: int):
    """Alg. 2 conditional node splitting (its body is missing, P:353 -> the
    reading in DESIGN.md §3 #24): walk the density-sorted tree top-down; a child c of a
    node with >= 2 children is an OUTLIER when its density lies strictly on the other side
    of the root density rho(rt) than the strict majority of its siblings' requests (each
    sibling subtree counts its |A| requests on the side of its own density; the dual
    scanner only needs each request on the correct side).  Relocating c
    duplicates the prefix it shares with its siblings, start(c) tokens ("potential
    recomputation waste"); it happens iff start(c) <= split_waste (the threshold t).  A
    relocated subtree is not searched further.  Returns group[r] (0 = stays, k >= 1 =
    the k-th relocated subtree in preorder)."""
    n = view["n_nodes"]
    cu_rt, mu_rt = root_key(view)
    kids = [[] for _ in range(n)]
    for i in range(n):
        par = int(view["node_parent"][i])
        if par >= 0:
            kids[par].append(i)

    def side(cu, mu):          # sign(rho - rho_rt) with rho = cu / mu, MU = 0 -> +inf
        if mu == 0:
            return 1 if cu > 0 or mu_rt > 0 else 0
        a, b = cu * mu_rt, cu_rt * mu
        return (a > b) - (a < b)

    group = np.zeros(w.n_req, dtype=np.int32)
    relocated = []

    def subtree_reqs(x):
        out, st = [], [x]
        while st:
            y = st.pop()
            out.extend(view["node_ends"][y])
            st.extend(kids[y])
        return out

    stack = [i for i in range(n) if int(view["node_parent"][i]) < 0][::-1]
    while stack:
        x = stack.pop()
        ch = kids[x]
        moved = set()
        if len(ch) >= 2:
            sides = {c: side(view["cu"][c], view["mu"][c]) for c in ch}
            for c in ch:
                up = sum(int(view["node_nreq"][o]) for o in ch if o != c and sides[o] > 0)
                down = sum(int(view["node_nreq"][o]) for o in ch if o != c and sides[o] < 0)
                ss = (up > down) - (up < down)
                sc = sides[c]
                if sc != 0 and ss != 0 and sc != ss and int(view["node_start"][c]) <= split_waste:
                    moved.add(c)
                    relocated.append(c)
        for c in reversed(ch):
            if c not in moved:
                stack.append(c)
    for k, c in enumerate(sorted(relocated), start=1):     # preorder ids = sorted node ids
        for r in subtree_reqs(c):
            group[r] = k
    return group


def build(w, rows_min: int = 128, min_sep_len: int = 128, force_class: int = 0,
          free_pages=None, split_waste: int = 0) -> dict:
    """Return the descriptor view (dict of numpy arrays + ints) for workload w.
    split_waste > 0 applies Alg. 2 (relocation_groups) to the sorted tree and rebuilds."""
    free = w.free_pages if free_pages is None else free_pages
    _validate(w, rows_min, min_sep_len, force_class, None if free is None else len(free))
    group = None
    if split_waste > 0:
        group = relocation_groups(w, build(w, rows_min, min_sep_len, force_class, free_pages), split_waste)
    root = _build_trie(w, group)
    nodes = _all_nodes(root)
    n_path = np.diff(w.tok_off).astype(object)
    p = [int(x) for x in w.prompt_len]
    d = [int(x) for x in w.out_len]

    # request sets A(N) (requests in the subtree) — post-order accumulation
    A = {}
    def collect(x):
        s = list(x.ends)
        for c in x.children.values():
            s.extend(collect(c))
        A[id(x)] = s
        return s
    for c in root.children.values():
        collect(c)

    maxP = {id(x): max(p[r] for r in A[id(x)]) for x in nodes}

    def clamp(v, lo, hi):
        return lo if v < lo else hi if v > hi else v

    def descendants(x):
        out, st = [], list(x.children.values())
        while st:
            y = st.pop()
            out.append(y)
            st.extend(y.children.values())
        return out

    Pm, H, L = int(w.model_params), int(w.hidden), int(w.layers)
    CU, MU = {}, {}
    for x in nodes:
        S = A[id(x)]
        mp = max(p[r] for r in S)
        G = 0
        y = x
        while y is not None and y is not root:            # X and its ancestors
            G += clamp(mp - y.start, 0, y.length)
            y = y.parent
        for y in descendants(x):
            G += clamp(maxP[id(y)] - y.start, 0, y.length)
        G += sum(max(0, p[r] - int(n_path[r])) for r in S)
        G += sum(d[r] for r in S)
        CU[id(x)] = 2 * Pm * G + 4 * H * L * sum(p[r] * p[r] for r in S)
        MU[id(x)] = sum(p[r] * d[r] + d[r] * (d[r] + 1) // 2 for r in S)
    minid = {id(x): min(A[id(x)]) for x in nodes}

    def cmp(a, b):
        ca, ma, cb, mb = CU[id(a)], MU[id(a)], CU[id(b)], MU[id(b)]
        def before(ca, ma, cb, mb):
            if ma == 0 and mb > 0:
                return True
            return ma > 0 and mb > 0 and ca * mb > cb * ma
        if before(ca, ma, cb, mb):
            return -1
        if before(cb, mb, ca, ma):
            return 1
        return -1 if minid[id(a)] < minid[id(b)] else 1

    order, dfs_req = [], []
    def visit(x):
        order.append(x)
        dfs_req.extend(sorted(x.ends))
        for c in sorted(x.children.values(), key=functools.cmp_to_key(cmp)):
            visit(c)
    for c in sorted(root.children.values(), key=functools.cmp_to_key(cmp)):
        visit(c)

    nid = {id(x): i for i, x in enumerate(order)}
    nn = len(order)
    R = w.n_req
    g = w.num_q_heads // w.num_kv_heads
    ps = w.page_size
    npages = [(x.length + ps - 1) // ps for x in order]
    page_off = np.zeros(nn + 1, dtype=np.int64)
    page_off[1:] = np.cumsum(npages)
    total_pages = int(page_off[-1])
    if free is None:
        page_table = np.arange(total_pages, dtype=np.int32)
    else:
        if len(free) < total_pages:
            raise BlendError(ENOSPC, "too few free pages")
        page_table = np.asarray(free[:total_pages], dtype=np.int32)
        if page_table.size and (page_table.min() < 0 or np.unique(page_table).size != total_pages):
            raise BlendError(EINVAL, "free page ids must be non-negative and distinct")

    q = [int(x) for x in w.q_len]
    req_big = [1 if q[r] * g >= rows_min else 0 for r in range(R)]
    node_class = np.zeros(nn, dtype=np.uint8)
    for i, x in enumerate(order):
        S = A[id(x)]
        if force_class == 2 or len(S) < 2:
            continue
        if force_class == 1:
            node_class[i] = 1
            continue
        small_rows = g * sum(q[r] for r in S if not req_big[r])
        if small_rows >= rows_min and x.length >= min_sep_len:
            node_class[i] = 1

    # request paths root -> end node
    end_node = {}
    for x in order:
        for r in x.ends:
            end_node[r] = x
    path_off = np.zeros(R + 1, dtype=np.int64)
    paths = []
    for r in range(R):
        chain, y = [], end_node[r]
        while y is not None and y is not root:
            chain.append(nid[id(y)])
            y = y.parent
        paths.append(chain[::-1])
        path_off[r + 1] = path_off[r] + len(chain)
    rank = np.zeros(R, dtype=np.int32)
    for k, r in enumerate(dfs_req):
        rank[r] = k

    def u128(v):
        return [v & 0xFFFFFFFFFFFFFFFF, v >> 64]

    return dict(
        n_req=R, n_nodes=nn,
        node_parent=np.array([nid[id(x.parent)] if x.parent is not root else -1 for x in order], dtype=np.int32),
        node_start=np.array([x.start for x in order], dtype=np.int32),
        node_len=np.array([x.length for x in order], dtype=np.int32),
        node_page_off=page_off,
        node_class=node_class,
        node_key_cu=np.array([u128(CU[id(x)]) for x in order], dtype=np.uint64).reshape(nn, 2),
        node_key_mu=np.array([u128(MU[id(x)]) for x in order], dtype=np.uint64).reshape(nn, 2),
        node_first_req=np.array([minid[id(x)] for x in order], dtype=np.int32),
        node_nreq=np.array([len(A[id(x)]) for x in order], dtype=np.int32),
        page_table=page_table,
        req_path_off=path_off,
        req_path_nodes=np.array([k for c in paths for k in c], dtype=np.int32),
        req_q_off=np.concatenate([[0], np.cumsum(q)]).astype(np.int64),
        req_class=np.array(req_big, dtype=np.uint8),
        req_dfs_rank=rank,
        req_global_id=(np.asarray(w.global_id, dtype=np.int64) if w.global_id is not None
                       else np.arange(R, dtype=np.int64)),
        req_group=(group if group is not None else np.zeros(R, dtype=np.int32)),
        # python-int keys for readability in tests
        cu=[CU[id(x)] for x in order], mu=[MU[id(x)] for x in order],
        dfs_order=np.array(dfs_req, dtype=np.int32),
        node_ends=[sorted(x.ends) for x in order],
    )


def dump(v, w) -> str:
    """Golden text dump (SPEC S:238 style), one line per node in id order:
    <2*depth spaces>#id start len tok=[first <=8 tokens] cu mu cls nreq ends=[...]"""
    lines = []
    depth = np.zeros(v["n_nodes"], dtype=np.int64)
    for i in range(v["n_nodes"]):
        par = int(v["node_parent"][i])
        depth[i] = 0 if par < 0 else depth[par] + 1
        r0 = int(v["node_first_req"][i])
        s, ln = int(v["node_start"][i]), int(v["node_len"][i])
        toks = w.path(r0)[s:s + min(ln, 8)]
        lines.append("%s#%d start=%d len=%d tok=[%s] cu=%d mu=%d cls=%s nreq=%d ends=[%s]" % (
            "  " * int(depth[i]), i, s, ln, ",".join(str(int(t)) for t in toks),
            v["cu"][i], v["mu"][i], "S" if v["node_class"][i] else "F",
            int(v["node_nreq"][i]), ",".join(str(x) for x in v["node_ends"][i])))
    return "\n".join(lines) + "\n"


# ---------------------------------------------------------------------------
# Density of a request set, hardware constants restored (P:87-96 cost model; P:309-315
# rho = Comp / Mem, rho(R) = (1 - s) T_comp / T_mem).  Used to check the C4 grid
# recipe's realised density and sharing and by the committed script
# that solves its request counts (scripts/solve_c4_counts.py).
# ---------------------------------------------------------------------------
def request_key(p: int, d: int, model_params: int, hidden: int, layers: int):
    """(CU, MU) of ONE request: P:89 Comp numerator (p + d) * P_model * 2 + p^2 * H * L * 4
    and P:93 Mem's exact sum sum_{i=1..d} (p + i) (hardware constants removed)."""
    return 2 * model_params * (p + d) + 4 * hidden * layers * p * p, p * d + d * (d + 1) // 2


def root_key(view):
    """(CU, MU) of the whole batch (the virtual root over the forest): top-level subtrees
    have disjoint closures and request sets, so their keys add."""
    tops = [i for i in range(view["n_nodes"]) if int(view["node_parent"][i]) < 0]
    return sum(view["cu"][i] for i in tops), sum(view["mu"][i] for i in tops)


def density(cu: int, mu: int, compute: float, bandwidth: float, kv_bytes_per_token: int) -> float:
    """rho = Comp / Mem = (CU / compute) / (MU * H_kv * L * 4 / bandwidth) (the
    4 = K and V at 2 bytes; reading #8: H_kv = Hkv * D)."""
    return (cu / compute) / (mu * kv_bytes_per_token / bandwidth) if mu else float("inf")


def sharing_ratio(w, view) -> float:
    """Prefix sharing ratio s of the batch read as the GEMM-token saving (SURVEY §8(d-4),
    P:141): 1 - CU_all / sum_r CU_r, CU_r the single-request key."""
    cu_all, _ = root_key(view)
    tot = sum(request_key(int(w.prompt_len[r]), int(w.out_len[r]), int(w.model_params), int(w.hidden),
                          int(w.layers))[0] for r in range(w.n_req))
    return 1.0 - cu_all / tot
