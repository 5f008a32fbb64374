"""Diagnostics (GPU): the bench's N-GPU data-parallel recipe with every rank's subtree
shard timed on this one GPU in turn — the per-rank step times whose max the N-GPU bench
would report.  Default (bench.py's mode): ONE global workload split into N shards, strong
scaling, reported as the projected speedup over the 1-GPU step; --weak: N copies.
Usage: python scripts/dp_shard_balance.py c4 2 4 8    |    ... --weak c2 2 4 8"""
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
import bench  # noqa: E402
import paper_2411_16102_b200 as B  # noqa: E402
from harness.run import build_tree, device_batch, subset  # noqa: E402

args = [a for a in sys.argv[1:] if a != "--weak"]
weak = "--weak" in sys.argv
name = args[0]
flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
t1 = None
for G in [1] + ([int(x) for x in args[1:]] or [2, 4, 8]):
    gw = bench.make_workload(name, G if weak else 1)
    req_shard = build_tree(gw, num_sms=148).shard(G)[0] if G > 1 else np.zeros(gw.n_req, np.int32)
    times = []
    for r in range(G):
        w = subset(gw, np.nonzero(req_shard == r)[0]) if G > 1 else gw
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
    if G == 1:
        t1 = float(t[0])
    tail = (f"weak-scaling efficiency vs the slowest rank {t.mean() / t.max():.3f}" if weak else
            f"projected strong-scaling speedup {t1 / t.max():.2f}x (efficiency {t1 / t.max() / G:.3f})")
    print(f"{name} x{G}: per-rank ms {np.round(t, 4).tolist()}  max {t.max():.4f}  mean {t.mean():.4f}  {tail}",
          flush=True)
