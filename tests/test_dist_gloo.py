"""Multi-process (gloo, world size 2) coverage of the data-parallel plumbing:
every rank builds the global tree through the C ABI, blend_shard assigns whole
subtrees, each rank builds its shard plan and executes it (CPU plan interpreter
standing in for the GPU), outputs are all-gathered and re-ordered by req_shard,
and the assembled result matches the oracle; timings are all-reduced with MAX."""
import os
import socket

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


def _worker(rank, port, name, resq):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=WORLD)
    try:
        from harness.run import build_tree, subset
        from tests.plan_sim import simulate
        from synth import workloads as W
        from tests.helpers import random_workload

        if name == "c1d":
            w = W.replicate(lambda seed: W.c1_tiny("d", "f32", seed=seed), WORLD, 1)
        else:
            w = random_workload(11, n_req=20, hq=4, hkv=2, max_seg=60)
        tree = build_tree(w)
        req_shard, _ = tree.shard(WORLD)
        mine = np.nonzero(req_shard == rank)[0]
        ws = subset(w, mine)
        out, lse, written, _ = simulate(ws, build_tree(ws))
        assert np.all(written == 1)
        # gather (padded) outputs over the process group
        rows = torch.tensor([out.shape[0]])
        dist.all_reduce(rows, op=dist.ReduceOp.MAX)
        pad = torch.zeros((int(rows.item()),) + out.shape[1:], dtype=torch.float64)
        pad[:out.shape[0]] = torch.from_numpy(out)
        gathered = [torch.zeros_like(pad) for _ in range(WORLD)]
        dist.all_gather(gathered, pad)
        t = torch.tensor([float(rank + 1)])
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        if rank == 0:
            # re-assemble in global request order
            q = w.q_len.astype(np.int64)
            qo = np.concatenate([[0], np.cumsum(q)])
            full = np.zeros((int(q.sum()),) + out.shape[1:])
            for g in range(WORLD):
                rs = np.nonzero(req_shard == g)[0]
                off = 0
                for r in rs:
                    full[qo[r]:qo[r + 1]] = gathered[g][off:off + q[r]].numpy()
                    off += q[r]
            from oracle import attention as A
            ref = A.attention_workload(w)
            err = max(float(np.max(np.abs(full[qo[r]:qo[r + 1]] - ref[r][0]))) for r in range(w.n_req))
            resq.put((err, float(t.item()), [int((req_shard == g).sum()) for g in range(WORLD)]))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("name", ["c1d", "random"])
def test_gloo_shard_gather(name):
    ctx = mp.get_context("spawn")
    q = ctx.SimpleQueue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, port, name, q)) for r in range(WORLD)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(timeout=300)
        assert p.exitcode == 0
    err, tmax, counts = q.get()
    assert err < 1e-10
    assert tmax == WORLD
    assert all(c > 0 for c in counts)
