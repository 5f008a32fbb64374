"""Diagnostics (GPU): per-CTA timeline of the dense kernel's first unit from globaltimer
stamps (blend_internal_set_trace).  Slots: 0 start, 1 setup done, 2 MMA sees Q, 3 first
K/V TMA issued, 8+2j S(j) seen by softmax A, 9+2j P(j) handed over, 4 epilogue start,
5 epilogue end, 6 CTA exit.  Usage: python scripts/trace_dense.py c2"""
import ctypes as C
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
import bench  # noqa: E402
import paper_2411_16102_b200 as B  # noqa: E402
from harness.run import device_batch  # noqa: E402

w = bench.make_workload(sys.argv[1] if len(sys.argv) > 1 else "c2")
db = device_batch(w, tree_kw=dict(num_sms=148))
for _ in range(3):
    db.run()
torch.cuda.synchronize()
tr = torch.zeros((297, 64), dtype=torch.int64, device="cuda")   # dense rows 0..147, streaming 148..295, counters 296
L = B.lib()
L.blend_internal_set_trace.argtypes = [C.c_void_p]
L.blend_internal_set_trace(tr.data_ptr())
db.run(flags=B.SERIALIZE)
torch.cuda.synchronize()
L.blend_internal_set_trace(None)
tall = tr.cpu().numpy()
if tall[296, 8] + tall[296, 9] > 0:
    print(f"softmax blocks (warp level): fast {tall[296, 8]}, slow {tall[296, 9]} "
          f"({100.0 * tall[296, 9] / (tall[296, 8] + tall[296, 9]):.1f} % slow)")
t = tall.astype(np.float64)[:148]
used = t[:, 0] > 0
t = t[used]
t0 = t[:, 0].min()
rel = np.where(t > 0, (t - t0) / 1e3, np.nan)   # us
names = {0: "start", 1: "setup", 2: "mma_q", 3: "tma0", 4: "epi0", 5: "epi1", 6: "exit", 60: "o_done", 61: "stored", 62: "ld_c0", 63: "st_c0"}
print(f"{w.name}: {used.sum()} CTAs, dense units {db.info['n_dense_units']}")
if not np.all(np.isnan(rel[:, 20])) and np.nanmax(rel[:, 20:40]) > 0:
    print("per-unit (BLEND_TRACE_UNITS): start / end of the k-th unit of a CTA (tile A)")
    for k in range(10):
        st, en = np.nanmedian(rel[:, 20 + 2 * k]), np.nanmedian(rel[:, 21 + 2 * k])
        print(f"  unit {k}: start {st:8.2f} end {en:8.2f}  ({en - st:6.2f} us)")
for k in list(range(7)) + [60, 62, 63, 61] + list(range(8, 20)):
    col = rel[:, k]
    if np.all(np.isnan(col)):
        continue
    nm = names.get(k, f"S{(k - 8) // 2}" if k % 2 == 0 else f"P{(k - 8) // 2}")
    print(f"{nm:>6}: median {np.nanmedian(col):8.2f} us  min {np.nanmin(col):8.2f}  max {np.nanmax(col):8.2f}")
