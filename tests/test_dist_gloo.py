"""Multi-process (gloo, world size 2) coverage of the multi-GPU plumbing that bench.py
runs over NCCL: harness/dp.py's shard_batch (global tree through the C ABI, blend_shard,
the rank's subtree shard), gather_rows (all-gather of out AND lse, re-assembly in global
request order by req_shard) and, for head parallelism, tp_heads / gather_heads.  Each
rank executes its own plan with the CPU plan interpreter (tests/plan_sim.py) standing in
for the GPU; rank 0 checks the assembled result against the fp64 oracle."""
import os
import socket
from dataclasses import replace

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

WORLD = 2


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _workload(name):
    from synth import workloads as W
    from tests.helpers import random_workload
    if name == "c1d":
        return W.replicate(lambda seed: W.c1_tiny("d", "f32", seed=seed), WORLD, 1)
    if name == "c1b_one_batch":
        return W.c1_tiny("b", "f32")
    return random_workload(11, n_req=20, hq=4, hkv=2, max_seg=60)


def _worker(rank, port, name, mode, resq):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=WORLD)
    try:
        from harness.dp import gather_heads, gather_rows, shard_batch, tp_heads
        from harness.run import build_tree
        from oracle import attention as A
        from tests.plan_sim import simulate

        gw = _workload(name)
        if mode == "dp":
            w, req_shard, _ = shard_batch(gw, WORLD, rank)
        else:
            gw = replace(gw, num_q_heads=4, num_kv_heads=2) if gw.num_kv_heads < 2 else gw
            hq, hkv, h0, kvh0 = tp_heads(gw, WORLD, rank)
            w = replace(gw, num_q_heads=hq, num_kv_heads=hkv, head0=h0, kv_head0=kvh0)
        out, lse, written, _ = simulate(w, build_tree(w))
        assert np.all(written == 1)
        o_t, l_t = torch.from_numpy(out), torch.from_numpy(lse)
        if mode == "dp":
            of, lf = gather_rows(o_t, l_t, gw, req_shard, WORLD, dist)
        else:
            of, lf = gather_heads(o_t, l_t, WORLD, dist)
        t = torch.tensor([float(rank + 1)])
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        if rank == 0:
            ref = A.attention_workload(gw)
            qo = np.concatenate([[0], np.cumsum(gw.q_len)])
            err = max(float(np.max(np.abs(of[qo[r]:qo[r + 1]].numpy() - O))) for r, (O, L) in ref.items())
            lerr = max(float(np.max(np.abs(lf[qo[r]:qo[r + 1]].numpy() - L))) for r, (O, L) in ref.items())
            counts = [int((req_shard == g).sum()) for g in range(WORLD)] if mode == "dp" else [w.num_q_heads] * 2
            resq.put((err, lerr, float(t.item()), counts))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("name,mode", [("c1d", "dp"), ("random", "dp"), ("c1b_one_batch", "dp"),
                                       ("random", "tp")])
def test_gloo_multi_rank(name, mode):
    ctx = mp.get_context("spawn")
    q = ctx.SimpleQueue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, port, name, mode, q)) for r in range(WORLD)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(timeout=300)
        assert p.exitcode == 0
    err, lerr, tmax, counts = q.get()
    assert err < 1e-10 and lerr < 1e-10
    assert tmax == WORLD
    assert all(c > 0 for c in counts)
