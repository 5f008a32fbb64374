"""Whole-workload run (NEXT-2, "all processed tokens ... divided by the total
processing time"): the dual-scanner batch former (blend_schedule_build) turns a whole offline
workload into its stream of blended batches; every k-th step (systematic sample) is
materialised as a step workload (each request's prompt prefix, then its generated tokens),
planned, filled and timed through blend_attention.  The sampled steps' times scaled by k
estimate the whole run's attention time (an unbiased estimator of the total for systematic
sampling); tokens are counted exactly over all steps.

Input plumbing only: the scheduling runs in libblend (host), the attention in libblend's
kernels.
"""
from __future__ import annotations

import time

import numpy as np

import paper_2411_16102_b200 as B
from harness.run import build_tree, device_batch
from synth.workloads import step_workload


def whole_run(w, mem_tokens: int, n_sample: int = 24, reps: int = 3, policy: int = B.SCHED_DUAL,
              tree_kw=None, chunk: int = 512, step_budget: int = 8192):
    import torch
    t0 = time.perf_counter()
    tree = build_tree(w)
    sched = tree.schedule(mem_tokens, chunk=chunk, step_budget=step_budget, policy=policy)
    host_s = time.perf_counter() - t0
    S = int(sched["n_steps"])
    so, req, nc, q = sched["step_off"], sched["req"], sched["n_cached"], sched["q"]
    step_tokens = np.add.reduceat(q.astype(np.int64), so[:-1]) if S else np.zeros(0, np.int64)
    k = max(1, S // n_sample)
    picks = list(range(k // 2, S, k))
    times, toks = [], []
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    for s in picks:
        a, b = int(so[s]), int(so[s + 1])
        sw = step_workload(w, req[a:b], nc[a:b], q[a:b], name=f"{w.name}_step{s}")
        db = device_batch(sw, tree_kw=tree_kw)
        db.run()                                             # warm-up (tensor maps, smem attributes)
        torch.cuda.synchronize()
        ts = []
        for _ in range(reps):
            ev0.record()
            db.run()
            ev1.record()
            torch.cuda.synchronize()
            ts.append(ev0.elapsed_time(ev1))
        times.append(float(np.median(ts)))
        toks.append(int(q[a:b].sum()))
        del db
    est_ms = float(np.sum(times)) * S / max(1, len(picks))
    return dict(
        n_steps=S, sampled_steps=len(picks), sample_stride=k, total_tokens=int(step_tokens.sum()),
        est_total_ms=est_ms, tokens_per_s=int(step_tokens.sum()) / (est_ms * 1e-3) if est_ms > 0 else None,
        sampled_tokens_per_s=float(np.sum(toks)) / (float(np.sum(times)) * 1e-3) if times else None,
        step_ms_median=float(np.median(times)) if times else None,
        sharing_vs_optimal=sched["cached_prompt_tokens"] / max(1, sched["optimal_cached_tokens"]),
        cached_prompt_tokens=int(sched["cached_prompt_tokens"]),
        optimal_cached_tokens=int(sched["optimal_cached_tokens"]),
        schedule_host_s=host_s, mem_tokens=mem_tokens, policy="dual" if policy == B.SCHED_DUAL else "dfs")
