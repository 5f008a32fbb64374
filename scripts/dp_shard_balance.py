"""Diagnostics (GPU): the bench's N-GPU data-parallel recipe (N copies of a workload,
blend_shard into N subtree shards) with every shard timed on this one GPU in turn —
the per-rank step times whose max the N-GPU bench would report (weak scaling).
Usage: python scripts/dp_shard_balance.py c2 2 4 8"""
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
import bench  # noqa: E402
import paper_2411_16102_b200 as B  # noqa: E402
from harness.run import build_tree, device_batch, subset  # noqa: E402

name = sys.argv[1]
flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
for G in [int(x) for x in sys.argv[2:]] or [2, 4, 8]:
    gw = bench.make_workload(name, G)
    req_shard, _ = build_tree(gw, num_sms=148).shard(G)
    times = []
    for r in range(G):
        w = subset(gw, np.nonzero(req_shard == r)[0])
        db = device_batch(w, tree_kw=dict(num_sms=148))
        for _ in range(3):
            db.run()
        ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(10)]
        for a, b in ev:
            B.l2_flush(flush)
            a.record()
            db.run()
            b.record()
        torch.cuda.synchronize()
        times.append(float(np.mean([a.elapsed_time(b) for a, b in ev])))
        del db
    t = np.array(times)
    print(f"{name} x{G}: per-rank ms {np.round(t, 4).tolist()}  max {t.max():.4f}  mean {t.mean():.4f}  "
          f"weak-scaling efficiency vs the slowest rank {t.mean() / t.max():.3f}")
