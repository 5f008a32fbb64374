"""Diagnostics (GPU): per-block ping-pong timeline of the dense kernel's first unit
(BLEND_TRACE_BLOCKS build of scripts/ab/dense_128key.cu: BLEND_SRC_OVERRIDE="dense.cu=$PWD/scripts/ab/dense_128key.cu"): for blocks j < 12, when each tile's softmax saw S_t(j)
(slot 8+2j tile A, 32+2j tile B) and handed P_t(j) over (9+2j / 33+2j).  Medians over
CTAs, microseconds from the CTA's first S.  Usage: BLEND_LIB=...libblend_tb.so python
scripts/trace_blocks.py c4"""
import ctypes as C
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
import bench  # noqa: E402
import paper_2411_16102_b200 as B  # noqa: E402
from harness.run import device_batch  # noqa: E402

w = bench.make_workload(sys.argv[1] if len(sys.argv) > 1 else "c4")
db = device_batch(w, tree_kw=dict(num_sms=148))
for _ in range(3):
    db.run()
torch.cuda.synchronize()
tr = torch.zeros((297, 64), dtype=torch.int64, device="cuda")
L = B.lib()
L.blend_internal_set_trace.argtypes = [C.c_void_p]
L.blend_internal_set_trace(tr.data_ptr())
db.run(flags=B.SERIALIZE)
torch.cuda.synchronize()
L.blend_internal_set_trace(None)
t = tr.cpu().numpy().astype(np.float64)[:148]
t = t[t[:, 8] > 0]
t0 = t[:, 8:9]
rel = np.where(t > 0, (t - t0) / 1e3, np.nan)
print(f"{w.name}: {len(t)} CTAs; per block j: tile A S seen / P out, tile B S seen / P out "
      "(median us from S_A(0)); softmax time = P - S")
for j in range(12):
    sa, pa, sb, pb = (np.nanmedian(rel[:, c]) for c in (8 + 2 * j, 9 + 2 * j, 32 + 2 * j, 33 + 2 * j))
    print(f"  j={j:2d}  A: {sa:7.3f} {pa:7.3f} ({pa - sa:5.3f})   B: {sb:7.3f} {pb:7.3f} ({pb - sb:5.3f})")
