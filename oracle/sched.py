"""Dual-scanner batch former oracle (NEXT-2) — independent re-implementation of
`blend_schedule_build` (must match it bit-exactly).  TEST INFRASTRUCTURE ONLY
(see oracle/__init__.py).

Follows PAPER §4.4 step by step; the readings for what the paper leaves open
are DESIGN.md §3 #25-#31.

 1. Scanner units ("scanning the leaf nodes ... from left to right and right to
    left"; P:7 subtree merging "reduces fragmentation"): in node-id (preorder) order, a
    node X whose children are ALL single-request leaves is one merged unit holding X's own
    ending requests and its children's, in DFS order; every other node with ending
    requests (and not inside a merged unit) is a unit of its ending requests.  A unit's
    density is its node's key (CU_X, MU_X).
 2. rho(rt) = the batch's root key (sum of the top-level keys).
 3. Memory partition (worked example P:379): with the left cursor on unit L
    and the right on unit R (L < R),
        M_L = floor(M (rho(rt) - rho_R) / (rho_L - rho_R)) clamped to [0, M] if rho_L > rho_R,
        else floor(M / 2);  M_R = M - M_L,
    exact rational arithmetic on the integer keys; recomputed whenever a cursor moves.
    When the cursors meet (L == R) the last unit is drawn by both sides.
 4. Continuous batching (§5): each step, side by side (left, then right),
    admit the side's next queued request while its footprint p + d (KV tokens, reading
    #27) fits the side's free memory M_side - used_side (a side with nothing active
    admits one request regardless, so one oversized request cannot deadlock it); a side
    whose queue empties moves its cursor inward (left: L + 1, right: R - 1) and the
    partition is recomputed; a cursor that would cross the other stops.
    On admission, the request's prompt prefix shared with an ACTIVE request or with the
    most recently completed request of either side (whose path stays cached: "only one
    path needs to be cached for reuse") — the longest common prefix, capped at
    that request's prompt length; active requests in admission order, then the left and
    the right side's last completed request, the first wins ties — is reused, not
    prefilled again (at least one prompt token is always computed): intra-batch prefix
    sharing ("exactly-once computation of shared prefixes"; reading #28).  The request then waits (no prefill entry) until its
    provider has materialised the reused prefix — in the same step at the earliest, the
    provider coming first in the batch.
 5. Step batch: every active request contributes one entry (admission order): while its
    prompt is not fully materialised, a chunked-prefill step of q = min(chunk, remaining,
    left-over prefill budget) tokens (P:15 chunked prefill; the per-step budget is served
    in admission order, a request with no budget left this step waits); afterwards decode
    steps j = 0..d-1 with q = 1 and cached path length p + j + 1 (the C4 snapshot
    convention, synth/workloads.c4_grid).  A request whose last decode ran is released
    after the step (its footprint returns to its side).
 6. Stop when nothing is active or queued, or after max_steps steps.
Outputs: per step [(request, n_cached_after_step, q)], the admission order, each
request's side, M_L per step, and the cached prompt tokens (for the sharing ratio vs the
optimum = sum_r p_r - distinct prompt tokens of the tree).
"""
from __future__ import annotations

from typing import List


def scanner_units(view) -> List[tuple]:
    """[(node id, [requests])] in scan order (step 1)."""
    n = view["n_nodes"]
    kids = [[] for _ in range(n)]
    for i in range(n):
        par = int(view["node_parent"][i])
        if par >= 0:
            kids[par].append(i)
    ends = view["node_ends"]
    merged = [False] * n
    inside = [False] * n
    units = []
    for x in range(n):                       # preorder
        par = int(view["node_parent"][x])
        if par >= 0 and (inside[par] or merged[par]):
            inside[x] = True
            continue
        ch = kids[x]
        if ch and all(not kids[c] and len(ends[c]) == 1 for c in ch):
            merged[x] = True
            reqs = list(ends[x]) + [ends[c][0] for c in ch]
            units.append((x, reqs))
        elif ends[x]:
            units.append((x, list(ends[x])))
    return units


def _lcp(view, w, a: int, b: int) -> int:
    """Shared path length of requests a and b = end of their deepest common node."""
    pa = [int(x) for x in view["req_path_nodes"][int(view["req_path_off"][a]):int(view["req_path_off"][a + 1])]]
    pb = [int(x) for x in view["req_path_nodes"][int(view["req_path_off"][b]):int(view["req_path_off"][b + 1])]]
    m = 0
    for x, y in zip(pa, pb):
        if x != y:
            break
        m = int(view["node_start"][x]) + int(view["node_len"][x])
    return m


def partition(M: int, cu_l, mu_l, cu_r, mu_r, cu_rt, mu_rt) -> int:
    """Step 3: M_L from the two equations of P:362-368 (exact, floor, clamped)."""
    from fractions import Fraction as F

    def rho(cu, mu):
        return None if mu == 0 else F(cu, mu)       # None = +infinity (d = 0)
    rl, rr, rt = rho(cu_l, mu_l), rho(cu_r, mu_r), rho(cu_rt, mu_rt)
    inf = lambda x: x is None                        # noqa: E731
    if inf(rr) or (not inf(rl) and rl <= rr):
        return M // 2
    if inf(rl):                                      # rho_L = inf: M_L -> 0 unless rt is inf too
        return M if inf(rt) else 0
    if inf(rt):
        return M
    ml = M * (rt - rr) / (rl - rr)
    return max(0, min(M, ml.numerator // ml.denominator))


def schedule(w, view, mem_tokens: int, chunk: int = 512, step_budget: int = 8192, policy: str = "dual",
             max_steps: int = 0):
    """The dual scanner (policy "dual"), or the tree's DFS order on one side with all of M
    ("dfs", the single-cursor reference for the sharing ratio)."""
    R = w.n_req
    p = [int(x) for x in w.prompt_len]
    d = [int(x) for x in w.out_len]
    if policy == "dfs":
        units = [(-1, [int(r) for r in view["dfs_order"]])]
    else:
        units = scanner_units(view)
    tops = [i for i in range(view["n_nodes"]) if int(view["node_parent"][i]) < 0]
    cu_rt, mu_rt = sum(view["cu"][i] for i in tops), sum(view["mu"][i] for i in tops)
    M = mem_tokens
    K = len(units)
    L, Rc = 0, K - 1
    met = K <= 1
    qL = list(units[0][1]) if K else []
    qR = list(units[K - 1][1]) if K > 1 else []
    shared = qL                                       # the queue both sides draw from once met

    def repartition():
        if met:
            return m_left                             # kept from before the cursors met
        xl, xr = units[L][0], units[Rc][0]
        return partition(M, view["cu"][xl], view["mu"][xl], view["cu"][xr], view["mu"][xr], cu_rt, mu_rt)

    m_left = M if met else 0
    m_left = repartition()
    used = [0, 0]
    active = []                          # [request, side, materialised prompt tokens, decodes done]
    order, side_of = [], [0] * R
    cached_total = 0
    steps, mleft_steps = [], []
    dep = {}                             # request -> (provider request, prefix it needs)
    last_done = [-1, -1]                 # the most recently completed request of each side
    while True:
        # ---- admission (step 4)
        for s in ((0,) if policy == "dfs" else (0, 1)):
            while True:
                q_s = shared if met else (qL if s == 0 else qR)
                if not q_s:
                    if met:
                        break
                    if s == 0 and L + 1 < Rc:
                        L += 1
                        qL = list(units[L][1])
                    elif s == 1 and Rc - 1 > L:
                        Rc -= 1
                        qR = list(units[Rc][1])
                    else:                             # the cursors meet on the other side's unit
                        shared = qR if s == 0 else qL
                        met = True
                    m_left = repartition()
                    continue
                cap = m_left if s == 0 else M - m_left
                r = q_s[0]
                fp = p[r] + d[r]
                if used[s] > 0 and used[s] + fp > cap:
                    break
                q_s.pop(0)
                cached, prov = 0, -1
                for a in [e[0] for e in active] + [x for x in last_done if x >= 0]:
                    c = min(_lcp(view, w, r, a), p[a])
                    if c > cached:
                        cached, prov = c, a
                cached = min(cached, max(0, p[r] - 1))
                if cached > 0:
                    dep[r] = (prov, cached)
                cached_total += cached
                used[s] += fp
                active.append([r, s, cached, 0])
                order.append(r)
                side_of[r] = s
        if not active:
            break
        # ---- one step (step 5)
        batch = []
        budget = step_budget
        mat_of = {e[0]: e for e in active}
        for e in active:
            r, s, mat, dec = e
            if mat < p[r]:
                if r in dep:
                    a, need = dep[r]
                    if a in mat_of and mat_of[a][2] < need:
                        continue                     # waiting for the provider's prefix
                q = min(chunk, p[r] - mat, budget)
                if q <= 0:
                    continue
                budget -= q
                e[2] = mat + q
                batch.append((r, mat + q, q))
            else:
                batch.append((r, p[r] + dec + 1, 1))
                e[3] = dec + 1
        steps.append(batch)
        mleft_steps.append(m_left)
        keep = []
        for e in active:
            r, s, mat, dec = e
            if mat >= p[r] and dec >= d[r]:
                used[s] -= p[r] + d[r]
                last_done[s] = r
            else:
                keep.append(e)
        active = keep
        if max_steps and len(steps) >= max_steps:
            break
    return dict(steps=steps, order=order, side=side_of, m_left=mleft_steps, cached_prompt_tokens=cached_total)


def optimal_cached_tokens(w, view) -> int:
    """P:480's optimum: every shared prompt token computed once = sum_r p_r - distinct
    prompt tokens (the unlimited-cache DFS order).  Prompt tokens of the tree: for node N,
    the prefix positions below max p over its requests (the c-2 clamp)."""
    p = [int(x) for x in w.prompt_len]
    n = view["n_nodes"]
    maxp = [0] * n
    for r in range(w.n_req):
        for k in range(int(view["req_path_off"][r]), int(view["req_path_off"][r + 1])):
            x = int(view["req_path_nodes"][k])
            maxp[x] = max(maxp[x], p[r])
    distinct = sum(max(0, min(maxp[x] - int(view["node_start"][x]), int(view["node_len"][x]))) for x in range(n))
    return sum(p) - distinct
