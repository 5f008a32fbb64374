#!/usr/bin/env python
"""bench.py — blended-batch attention tokens/s on B200 (BASELINE.json metric).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--workload c2|c3|c5|c1b_bf16|...]
                    [--impl ours|reference] [--path auto|generic|no_tcgen05]

One step = one blend_attention call (dense tcgen05 pass + streaming pass + LSE
merge) over the whole blended batch of the workload, one layer, inputs resident
in HBM.  Default workload = configs[1] (C2: Llama-3.1-8B shapes, decode batch
256 over a shared ~1K MMLU-like prefix).  Its working set (113 MB) fits in L2,
so L2 is flushed (256 MB write) between timed steps.

N > 1 (torchrun): weak scaling — the global batch is N independent copies of the
recipe (distinct system prompts); every rank builds the global tree, blend_shard
splits it 2N-block-fold into N subtree shards, each rank runs its shard.  No KV
crosses GPUs; NCCL only all-reduces the timings (max over ranks) and, outside
the timed region, all-gathers the outputs.

--impl reference: the fp64 oracle (oracle/attention.py) on the host cores, on a
bounded sample of the same workload each step (the paper publishes no attention
number; BASELINE.json "published" is empty).
"""
from __future__ import annotations

import argparse
import json
import os
import subprocess
import sys
import threading
import time

os.environ.setdefault("OMP_NUM_THREADS", "1")
os.environ.setdefault("OPENBLAS_NUM_THREADS", "1")
os.environ.setdefault("MKL_NUM_THREADS", "1")

import numpy as np  # noqa: E402

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "blended-batch attention tokens/s"
PEAKS_FALLBACK = {"hbm_gbs": 6650.0, "bf16_tflops": 1590.0, "bf16_tflops_sustained": 1400.0}


def load_peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        d = json.load(open(p))
        d["_source"] = "measured (MEASURED_PEAKS.json)"
        return d
    d = dict(PEAKS_FALLBACK)
    d["_source"] = "fallback (B200_PROFILING.md)"
    return d


PROFILE_TAG = "r1h"   # profiles/<tag>_ncu.json: ncu --set full captures of this code's kernels


def ncu_traffic(workload: str, kernel: str):
    """dram__bytes_read.sum + dram__bytes_write.sum of one launch of `kernel` on
    `workload` from the committed ncu --set full capture (profiles/), or None."""
    p = os.path.join(ROOT, "profiles", f"{PROFILE_TAG}_ncu.json")
    try:
        full = json.load(open(p))["full"]
    except (OSError, ValueError, KeyError):
        return None, None
    d = full.get(f"{workload}_{kernel}")
    if not d or "traffic_bytes" not in d:
        return None, None
    return float(d["traffic_bytes"]), f"profiles/{PROFILE_TAG}_ncu.json [{workload}_{kernel}]"


def make_workload(name: str, n_copies: int = 1):
    from synth import workloads as W
    recipes = {"c2": (W.c2_mmlu_decode, 2), "c3": (W.c3_burst_openvid, 3), "c5": (W.c5_70b_32k, 5)}
    if name in recipes:
        fn, seed = recipes[name]
        if n_copies == 1:
            return fn(seed=seed)
        return W.replicate(fn, n_copies, seed)
    if n_copies != 1:
        raise SystemExit(f"workload {name} has no multi-copy recipe")
    return W.by_name(name)


class ClockSampler:
    """nvidia-smi clocks + throttle reasons sampled during the timed region."""
    Q = ("clocks.sm,clocks.max.sm,clocks_event_reasons.active,clocks_event_reasons.hw_slowdown,"
         "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
         "clocks_event_reasons.sw_power_cap")

    def __init__(self, index: int):
        self.index = index
        self.rows = []
        self.proc = None

    def start(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.Q}", "--format=csv,noheader,nounits",
                 "-lms", "50"], stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except (FileNotFoundError, OSError):
            self.proc = None

    def _read(self):
        for line in self.proc.stdout:
            self.rows.append([x.strip() for x in line.split(",")])

    def stop(self):
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"], "samples": 0}
        time.sleep(0.12)
        self.proc.terminate()
        try:
            self.proc.wait(timeout=2)
        except subprocess.TimeoutExpired:
            self.proc.kill()
        rows = [r for r in self.rows if len(r) >= 7]
        sm = [float(r[0]) for r in rows if r[0].replace(".", "").isdigit()]
        mx = [float(r[1]) for r in rows if r[1].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[k] for r in rows for k in range(4) if r[3 + k].lower() == "active"})
        return {"sm_mhz": float(np.median(sm)) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": reasons, "samples": len(rows)}


def oracle_sample(w, budget_flops: float, seed: int = 0):
    """Stratified request sample (BIG/SMALL, shortest/longest contexts, random) whose
    F_alg is about budget_flops; returns sorted request indices."""
    g = w.num_q_heads // w.num_kv_heads
    n = np.diff(w.tok_off).astype(np.int64)
    q = w.q_len.astype(np.int64)
    f = 4 * w.head_dim * w.num_q_heads * (q * (n - q) + q * (q + 1) // 2)
    big = np.nonzero(q * g >= 128)[0]
    small = np.nonzero(q * g < 128)[0]
    rng = np.random.default_rng(seed)
    order = []
    for grp in (big, small):
        if len(grp):
            srt = grp[np.argsort(n[grp])]
            order += [int(srt[0]), int(srt[-1])]
    order += [int(x) for x in rng.permutation(w.n_req)]
    pick, tot = [], 0.0
    seen = set()
    for r in order:
        if r in seen:
            continue
        if tot >= budget_flops and len(pick) >= 2:
            break
        seen.add(r)
        pick.append(r)
        tot += float(f[r])
    return sorted(pick), f


def _oracle_worker(args):
    (w, reqs) = args
    from oracle import attention as A
    t = 0.0
    for r in reqs:
        K, Vv, Q = A.request_inputs(w, r)        # materialisation excluded (GPU starts from a resident cache)
        t0 = time.perf_counter()
        A.attention_request(K, Vv, Q, int(w.q_len[r]))
        t += time.perf_counter() - t0
    return t


def time_oracle(w, reqs, cores):
    import multiprocessing as mp
    chunks = [reqs[i::cores] for i in range(cores)]
    chunks = [c for c in chunks if c]
    ctx = mp.get_context("fork")
    with ctx.Pool(len(chunks)) as pool:
        t0 = time.perf_counter()
        per = pool.map(_oracle_worker, [(w, c) for c in chunks])
        wall = time.perf_counter() - t0
    # parallel attention-math time = the slowest worker's math time
    return max(per), wall


def cpu_baseline(w, budget_s=15.0):
    cores = len(os.sched_getaffinity(0))
    # calibrate: ~1 GFLOP/s per core for fp64 einsum is conservative
    reqs, f = oracle_sample(w, budget_flops=budget_s * cores * 1.0e9)
    t_math, wall = time_oracle(w, reqs, cores)
    reps = 1
    while t_math * reps < 0.3 * budget_s and reps < 64:   # small workloads: repeat for a stable time
        t2, _ = time_oracle(w, reqs, cores)
        t_math = (t_math * reps + t2) / (reps + 1)
        reps += 1
    f_s = float(f[reqs].sum())
    f_all = float(f.sum())
    t_full = t_math * f_all / f_s
    return {"value": w.sum_q / t_full, "unit": "tokens/s", "cores": cores, "kind": "oracle",
            "sample": f"{len(reqs)} of {w.n_req} requests (stratified), fp64 numpy, "
                      f"{t_math:.3f} s math per pass on {cores} cores (mean of {reps} passes); "
                      f"extrapolated by F_alg share {f_s / f_all:.4f}",
            "measured_s": t_math, "extrapolated_step_s": t_full}


def run_reference(args):
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return 0
    w = make_workload(args.workload)
    cores = len(os.sched_getaffinity(0))
    steps = args.steps + args.warmup
    budget = max(1.0, 90.0 / max(1, steps))          # seconds of CPU work per step
    tot_t = tot_tok = 0.0
    sample_desc = None
    for s in range(steps):
        reqs, f = oracle_sample(w, budget_flops=budget * cores * 1.0e9, seed=s)
        t_math, _ = time_oracle(w, reqs, cores)
        if s >= args.warmup:
            tot_t += t_math
            tot_tok += float(w.q_len[reqs].sum())
        sample_desc = f"{len(reqs)} of {w.n_req} requests per step (stratified, seed=step)"
    value = tot_tok / tot_t
    line = {"metric": METRIC, "value": value, "unit": "tokens/s", "impl": "reference",
            "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": 1e3 * tot_t / args.steps, "higher_is_better": True, "scaling": "weak",
            "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": {"workload": w.name, "requests": w.n_req, "query_tokens": int(w.sum_q),
                       "heads": f"{w.num_q_heads}/{w.num_kv_heads}x{w.head_dim}", "page_size": w.page_size,
                       "parallelism": "host cores (fp64 oracle)"},
            "cpu_baseline": {"value": value, "unit": "tokens/s", "cores": cores, "kind": "oracle",
                             "sample": sample_desc},
            "e2e": {"value": value, "unit": "tokens/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)
    return 0


def run_ours(args):
    import torch
    import torch.distributed as dist

    import paper_2411_16102_b200 as B
    from harness.run import build_tree, device_batch, pass_work, subset, work_counts

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if world != args.gpus:
        raise SystemExit(f"--gpus {args.gpus} but WORLD_SIZE={world}")
    torch.cuda.set_device(local)
    if world > 1:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    B.lib()
    path = {"auto": B.PATH_AUTO, "generic": B.PATH_GENERIC, "no_tcgen05": B.PATH_NO_TCGEN05}[args.path]
    tree_kw = dict(num_sms=torch.cuda.get_device_properties(local).multi_processor_count,
                   dense_split=args.dense_split, split_tokens=args.split_tokens)

    t0 = time.perf_counter()
    if args.tp:
        # NEXT-4: head-parallel replicas — every rank runs the whole
        # batch for its Hkv/N kv heads and their query-head groups (no exchange inside
        # attention); strong scaling of one batch.  Synthetic values use local head indices.
        from dataclasses import replace as _replace
        gw = make_workload(args.workload, 1)
        tpn = args.tp_ranks if args.tp_ranks else world   # --tp-ranks: one rank's slice of a wider TP group
        if gw.num_kv_heads % tpn:
            raise SystemExit(f"--tp: {gw.num_kv_heads} kv heads do not split over {tpn} ranks")
        w = _replace(gw, num_q_heads=gw.num_q_heads // tpn, num_kv_heads=gw.num_kv_heads // tpn,
                     name=f"{gw.name}_tp{tpn}_rank{rank}")
    else:
        gw = make_workload(args.workload, world)
        if world > 1:
            gtree = build_tree(gw, **tree_kw)
            req_shard, _ = gtree.shard(world)
            w = subset(gw, np.nonzero(req_shard == rank)[0], name=f"{gw.name}_shard{rank}")
        else:
            w = gw
    db = device_batch(w, tree_kw=tree_kw)
    host_s = time.perf_counter() - t0
    view = db.view
    F, Bytes, KVb = work_counts(w, view)
    pw = pass_work(w, view)
    info = db.info
    stream = torch.cuda.current_stream()
    flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
    do_flush = not args.no_flush

    for _ in range(args.warmup):
        db.run(path=path)
    torch.cuda.synchronize()

    K = args.steps
    def mk_events(n, m):
        evs = [[torch.cuda.Event(enable_timing=True) for _ in range(m)] for _ in range(n)]
        for row in evs:       # torch creates CUDA events lazily: materialise the handles
            for e in row:
                e.record(stream)
        return evs

    # ---- timed region: K whole steps (dense || streaming via PDL, then merge), events at the ends
    ev = mk_events(K, 2)
    # ---- per-pass breakdown: K serialised steps with events between the passes (roofline)
    evp = mk_events(K, 4)
    torch.cuda.synchronize()
    clocks = ClockSampler(local)
    clocks.start()
    time.sleep(0.2)
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    for k in range(K):
        if do_flush:
            B.l2_flush(flush)
        db.run(path=path, events=[ev[k][0], None, None, ev[k][1]])
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    clk = clocks.stop()
    for k in range(K):
        if do_flush:
            B.l2_flush(flush)
        db.run(path=path, events=evp[k], flags=B.SERIALIZE)
    torch.cuda.synchronize()
    t_step = [ev[k][0].elapsed_time(ev[k][1]) for k in range(K)]
    t_ser = [evp[k][0].elapsed_time(evp[k][3]) for k in range(K)]
    t_dense = [evp[k][0].elapsed_time(evp[k][1]) for k in range(K)]
    t_stream = [evp[k][1].elapsed_time(evp[k][2]) for k in range(K)]
    t_merge = [evp[k][2].elapsed_time(evp[k][3]) for k in range(K)]
    ms = float(np.mean(t_step))
    loc = torch.tensor([ms, float(np.mean(t_dense)), float(np.mean(t_stream)), float(np.mean(t_merge)),
                        float(np.mean(t_ser))], dtype=torch.float64, device="cuda")
    tok = torch.tensor([float(w.sum_q)], dtype=torch.float64, device="cuda")
    if world > 1:
        dist.all_reduce(loc, op=dist.ReduceOp.MAX)
        if not args.tp:   # TP: every rank works on the same tokens (its share of the heads)
            dist.all_reduce(tok, op=dist.ReduceOp.SUM)
    ms, md, mst, mm, mser = loc.tolist()
    total_tok = tok.item()
    value = total_tok / (ms * 1e-3)

    # ---- e2e through the public API: every step copies its Q in from pinned host memory
    # and its out + lse back.  Copies run on their own streams, double-buffered, so step
    # k's device->host read overlaps step k+1's attention and step k+2's host->device copy
    # (events order each buffer set: H2D -> attention -> D2H -> next H2D into the set).
    q_host = torch.empty(db.q.shape, dtype=db.q.dtype, pin_memory=True)
    q_host.copy_(db.q)
    io_bytes = 2 * db.q.numel() * db.q.element_size()
    NB = 4 if io_bytes < (256 << 20) else 2   # buffer sets in flight
    out_host = [torch.empty(db.out.shape, dtype=db.out.dtype, pin_memory=True) for _ in range(NB)]
    lse_host = [torch.empty(db.lse.shape, dtype=db.lse.dtype, pin_memory=True) for _ in range(NB)]
    qd = [db.q] + [torch.empty_like(db.q) for _ in range(NB - 1)]
    od = [db.out] + [torch.empty_like(db.out) for _ in range(NB - 1)]
    ld = [db.lse] + [torch.empty_like(db.lse) for _ in range(NB - 1)]
    # L2: a flush kernel on the compute stream would sit inside this timed region, so the
    # e2e steps instead use inputs larger than L2 — KV caches under 256 MB are rotated
    # over 3 copies (each step's cache was last touched two steps earlier, with >= 2x its
    # size of other traffic in between)
    kv_bytes = 2 * db.k_cache.numel() * db.k_cache.element_size()
    nrot = 3 if kv_bytes < (256 << 20) else 1
    kc = [db.k_cache] + [db.k_cache.clone() for _ in range(nrot - 1)]
    vc = [db.v_cache] + [db.v_cache.clone() for _ in range(nrot - 1)]
    s_h2d, s_d2h = torch.cuda.Stream(), torch.cuda.Stream()
    ev_h2d = [torch.cuda.Event() for _ in range(NB)]
    ev_cmp = [torch.cuda.Event() for _ in range(NB)]
    ev_d2h = [torch.cuda.Event() for _ in range(NB)]
    e2e_t0, e2e_t1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    # head start: the device sleeps (outside the timed region) while the host enqueues the
    # K steps, so the events time the device pipeline, not the Python loop that feeds it
    torch.cuda._sleep(int(2.0e9 * max(2e-3, K * 150e-6)))
    e2e_t0.record(stream)
    s_h2d.wait_event(e2e_t0)
    s_d2h.wait_event(e2e_t0)
    for k in range(K):
        b = k % NB
        with torch.cuda.stream(s_h2d):
            if k >= NB:
                s_h2d.wait_event(ev_d2h[b])            # set b's previous result has left the device
            qd[b].copy_(q_host, non_blocking=True)
            ev_h2d[b].record(s_h2d)
        stream.wait_event(ev_h2d[b])
        B.attention(qd[b], kc[k % nrot], vc[k % nrot], db.plan, od[b], ld[b], db.ws,
                    n_cache_pages=db.n_cache_pages, path=path, stream=stream)
        ev_cmp[b].record(stream)
        with torch.cuda.stream(s_d2h):
            s_d2h.wait_event(ev_cmp[b])
            out_host[b].copy_(od[b], non_blocking=True)
            lse_host[b].copy_(ld[b], non_blocking=True)
            ev_d2h[b].record(s_d2h)
    for b in range(min(K, NB)):
        stream.wait_event(ev_d2h[b])
    e2e_t1.record(stream)
    torch.cuda.synchronize()
    e2e_ms = torch.tensor([e2e_t0.elapsed_time(e2e_t1) / K], dtype=torch.float64, device="cuda")
    if world > 1:
        dist.all_reduce(e2e_ms, op=dist.ReduceOp.MAX)
    e2e_ms = e2e_ms.item()
    h2d = db.q.numel() * db.q.element_size()
    d2h = db.out.numel() * db.out.element_size() + db.lse.numel() * db.lse.element_size()
    # the copied-back result of the last step equals the device result of the same input
    e2e_match = bool(torch.equal(out_host[(K - 1) % NB], od[0].cpu()))

    # ---- output gather over NVLink (timed separately, not in the metric)
    gather_ms = None
    if world > 1:
        rows = torch.tensor([db.out.shape[0]], device="cuda")
        dist.all_reduce(rows, op=dist.ReduceOp.MAX)
        pad = torch.zeros((int(rows.item()),) + tuple(db.out.shape[1:]), dtype=db.out.dtype, device="cuda")
        pad[:db.out.shape[0]] = db.out
        allo = torch.empty((world,) + tuple(pad.shape), dtype=pad.dtype, device="cuda")
        g0, g1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        dist.barrier()
        g0.record()
        dist.all_gather_into_tensor(allo, pad)
        g1.record()
        torch.cuda.synchronize()
        gather_ms = g0.elapsed_time(g1)

    # our kernels per timed step: dense + streaming (+ merge: only off the arrival-merge
    # path, i.e. the generic executor) + the L2 flush between steps
    arrival = False   # BLEND_ARRIVAL_MERGE is opt-in; the bench runs the default path
    launches_per_step = int(info["n_dense_units"] > 0) + int(info["n_stream_units"] > 0) + \
        int(info["n_merge_tokens"] > 0 and not arrival) + int(do_flush)

    # ---- roofline of the dominant kernel (per launch, CUDA events on the launching stream)
    peaks = load_peaks()
    burst = ms < 100.0
    if md >= mst:
        tf = pw["dense_flops"] / (md * 1e-3) / 1e12
        peak = peaks["bf16_tflops"] if burst else peaks.get("bf16_tflops_sustained", peaks["bf16_tflops"])
        traffic, tsrc = ncu_traffic(args.workload, "dense_kernel") if path == B.PATH_AUTO else (None, None)
        roof = {"kernel": "dense (tcgen05)" if path == B.PATH_AUTO else "dense (generic executor)",
                "bound": "tensor", "achieved": tf, "peak": peak, "unit": "TFLOP/s", "frac": tf / peak,
                "traffic": traffic, "traffic_source": tsrc, "algorithmic_per_launch": pw["dense_flops"],
                "algorithmic_bytes_per_launch": pw["dense_bytes"],
                "peak_source": peaks["_source"] + (" burst" if burst else " sustained")}
    else:
        gbs = pw["stream_bytes"] / (mst * 1e-3) / 1e9
        peak = peaks["hbm_gbs"]
        traffic, tsrc = ncu_traffic(args.workload, "streamw_kernel") if path == B.PATH_AUTO else (None, None)
        roof = {"kernel": "stream", "bound": "hbm", "achieved": gbs, "peak": peak, "unit": "GB/s",
                "frac": gbs / peak, "traffic": traffic, "traffic_source": tsrc,
                "algorithmic_per_launch": pw["stream_bytes"], "peak_source": peaks["_source"]}

    line = None
    if rank == 0:
        cpu = None
        if world == 1 and not args.no_cpu_baseline:
            try:
                cpu = cpu_baseline(w)
            except Exception as e:  # noqa: BLE001
                cpu = {"value": None, "unit": "tokens/s", "cores": len(os.sched_getaffinity(0)),
                       "kind": "oracle", "sample": f"failed: {e}"}
        line = {
            "metric": METRIC, "value": value, "unit": "tokens/s", "n_gpus": world, "steps": K,
            "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": True,
            "scaling": "strong" if args.tp else "weak",
            "vs_baseline": None, "dtype": "bf16" if w.kv_dtype == "bf16" else "f32", "data": "synthetic",
            "config": {"workload": gw.name, "requests": gw.n_req, "query_tokens": int(total_tok),
                       "heads": f"{gw.num_q_heads}/{gw.num_kv_heads}x{gw.head_dim}"
                                + (f" (per rank {w.num_q_heads}/{w.num_kv_heads})" if args.tp else ""),
                       "page_size": w.page_size,
                       "parallelism": (f"tp{world} (kv heads)" if args.tp else f"dp{world} (subtree shards)")
                       if world > 1 else ((f"one rank of tp{args.tp_ranks} (kv heads)" if args.tp_ranks
                                           else "tp1 (kv heads)") if args.tp else "single GPU"),
                       "l2": "flushed (256 MB write) between timed steps" if do_flush else "not flushed",
                       "path": args.path},
            "clocks": clk,
            "e2e": {"value": total_tok / (e2e_ms * 1e-3), "unit": "tokens/s", "h2d_bytes_per_step": h2d,
                    "d2h_bytes_per_step": d2h, "ms_per_step": e2e_ms,
                    "note": "blend_attention with Q copied in from pinned host memory and out + lse copied "
                            "back every step; copies on side streams, NB buffer sets (step k's D2H "
                            "overlaps step k+1's attention and step k+2's upload)", "buffer_sets": NB, "output_matches_device": e2e_match,
                    "l2": (f"KV rotated over {nrot} copies ({nrot * kv_bytes >> 20} MB > L2), no flush in the "
                           "timed region" if nrot > 1 else "inputs larger than L2, no flush in the timed region")},
            "gpu_launches": launches_per_step * K,
            "roofline": roof,
            "cpu_baseline": cpu,
            "passes_ms": {"dense": md, "stream": mst, "merge": mm, "serialized_step": mser,
                          "note": "per-pass times from K extra steps run with BLEND_SERIALIZE (dense grid on "
                                  "every SM); the timed steps overlap the dense and streaming passes (PDL), "
                                  "with the dense grid capped by the planner when both passes are large"},
            "work": {"F_alg": F, "B_alg": Bytes, "kv_bytes": KVb, **pw,
                     "whole_step_roofline_frac_measured": max(F / (load_peaks()["bf16_tflops"] * 1e12),
                                                              Bytes / (load_peaks()["hbm_gbs"] * 1e9)) / (ms * 1e-3)},
            "plan": info,
            "host_build_s": host_s,
            "gather_ms": gather_ms,
        }
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.barrier()
        dist.destroy_process_group()
    return 0


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=50)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--workload", default="c2")
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--path", default="auto", choices=["auto", "generic", "no_tcgen05"])
    ap.add_argument("--no-flush", action="store_true")
    ap.add_argument("--dense-split", type=int, default=0, help="dense split-KV factor (0 = planner auto)")
    ap.add_argument("--split-tokens", type=int, default=0, help="streaming split-KV chunk (0 = auto)")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--tp", action="store_true",
                    help="head-parallel replicas (NEXT-4): each rank takes Hkv/N kv heads of the whole batch")
    ap.add_argument("--tp-ranks", type=int, default=0,
                    help="with --tp on one GPU: time one rank's slice of a TP group of this size "
                         "(the line's value is that rank's tokens/s, not a group total)")
    args = ap.parse_args()
    if args.warmup < 3:
        raise SystemExit("--warmup must be >= 3")
    if args.impl == "reference":
        return run_reference(args)
    return run_ours(args)


if __name__ == "__main__":
    sys.exit(main())
