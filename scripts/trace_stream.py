"""Diagnostics (GPU): streaming-pass timeline (warp 0 of each CTA) from globaltimer
stamps.  Slots: 0 CTA start, 60 first unit index, per unit u: 2+4u start, 3+4u first
stage data, 4+4u KV loop end, 5+4u unit end.  Times relative to the dense kernel's
first CTA start.  Usage: python scripts/trace_stream.py c2"""
import ctypes as C
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
import bench  # noqa: E402
import paper_2411_16102_b200 as B  # noqa: E402
from harness.run import device_batch  # noqa: E402

w = bench.make_workload(sys.argv[1] if len(sys.argv) > 1 else "c2")
flags = int(sys.argv[2]) if len(sys.argv) > 2 else 0
db = device_batch(w, tree_kw=dict(num_sms=148))
for _ in range(3):
    db.run()
torch.cuda.synchronize()
tr = torch.zeros((297, 64), dtype=torch.int64, device="cuda")
tr[296, 0] = 2**62   # merge kernel: first start (atomicMin), last end (atomicMax)
L = B.lib()
L.blend_internal_set_trace.argtypes = [C.c_void_p]
L.blend_internal_set_trace(tr.data_ptr())
db.run(flags=flags)
torch.cuda.synchronize()
L.blend_internal_set_trace(None)
t = tr.cpu().numpy().astype(np.float64)
t0 = t[:148, 0][t[:148, 0] > 0].min() if (t[:148, 0] > 0).any() else t[148:, 0][t[148:, 0] > 0].min()
s = t[148:296]
s = s[s[:, 0] > 0]
rel = np.where(s > 0, (s - t0) / 1e3, np.nan)
print(f"{w.name}: {len(s)} streaming CTAs (flags={flags}); dense CTAs {(t[:148, 0] > 0).sum()}")
print(f"  CTA start: median {np.nanmedian(rel[:, 0]):.2f} min {np.nanmin(rel[:, 0]):.2f} max {np.nanmax(rel[:, 0]):.2f} us")
for u in range(14):
    cols = [2 + 4 * u, 3 + 4 * u, 4 + 4 * u, 5 + 4 * u]
    if np.all(np.isnan(rel[:, cols[0]])):
        break
    st, fd, ke, en = (np.nanmedian(rel[:, c]) for c in cols)
    n = int(np.sum(~np.isnan(rel[:, cols[0]])))
    print(f"  unit {u}: start {st:7.2f} data {fd:7.2f} kv_end {ke:7.2f} end {en:7.2f}  ({n} CTAs)")
if not np.all(np.isnan(rel[:, 36])):
    print("  stages 4..11 (ring 0): TMA issue", [round(float(np.nanmedian(rel[:, 52 + k])), 2) for k in range(8)])
    print("                         data      ", [round(float(np.nanmedian(rel[:, 36 + k])), 2) for k in range(8)])
    print("                         freed     ", [round(float(np.nanmedian(rel[:, 44 + k])), 2) for k in range(8)])
last = np.nanmax(rel[:, 2:30], axis=1)
d6 = t[:148, 6][t[:148, 6] > 0]
if len(d6):
    print(f"  dense CTA exit: median {np.median((d6 - t0) / 1e3):.2f} max {np.max((d6 - t0) / 1e3):.2f} us")
m0, m1 = t[296, 0], t[296, 1]
if 0 < m0 < 2**62:
    print(f"  merge kernel: first start {(m0 - t0) / 1e3:.2f} us, last end {(m1 - t0) / 1e3:.2f} us")
print(f"  warp-0 last stamp: median {np.nanmedian(last):.2f} max {np.nanmax(last):.2f}")
