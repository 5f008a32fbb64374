"""Diagnostics (GPU): per-pass times (serialised, CUDA events) and plan shape of rank r's
subtree shard of a workload split over G GPUs (bench.py's strong-scaling DP), timed on
this one GPU.  Usage: python scripts/dp_rank_passes.py c5 8 [rank] [--dense-split S]"""
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
import bench  # noqa: E402
import paper_2411_16102_b200 as B  # noqa: E402
from harness.run import build_tree, device_batch, subset  # noqa: E402

args = [a for a in sys.argv[1:] if not a.startswith("--")]
name, G = args[0], int(args[1])
rank = int(args[2]) if len(args) > 2 else 0
kw = dict(num_sms=148)
if "--dense-split" in sys.argv:
    kw["dense_split"] = int(sys.argv[sys.argv.index("--dense-split") + 1])
gw = bench.make_workload(name)
req_shard = build_tree(gw, num_sms=148).shard(G)[0] if G > 1 else np.zeros(gw.n_req, np.int32)
w = subset(gw, np.nonzero(req_shard == rank)[0])
db = device_batch(w, tree_kw=kw)
import ctypes as C  # noqa: E402
f = B.lib().blend_internal_dense_ctas
f.restype, f.argtypes = C.c_int32, [C.c_void_p]
print(f"{name} rank {rank}/{G}: {w.n_req} requests, plan {db.info}, dense_ctas {f(db.tree.handle)}")
flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
for _ in range(3):
    db.run()
res = {"overlapped": [], "dense": [], "stream": [], "merge": []}
for _ in range(10):
    B.l2_flush(flush)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    db.run()
    e1.record()
    torch.cuda.synchronize()
    res["overlapped"].append(e0.elapsed_time(e1))
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(4)]
    for e in ev:        # torch creates CUDA events lazily: materialise the handles
        e.record()
    B.l2_flush(flush)
    db.run(events=ev, flags=B.SERIALIZE)
    torch.cuda.synchronize()
    res["dense"].append(ev[0].elapsed_time(ev[1]))
    res["stream"].append(ev[1].elapsed_time(ev[2]))
    res["merge"].append(ev[2].elapsed_time(ev[3]))
print({k: round(float(np.median(v)), 4) for k, v in res.items()})
