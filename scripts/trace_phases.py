"""Diagnostics (GPU): mean clock cycles per softmax phase of tile A's first unit
(BLEND_TRACE_PHASES build of scripts/ab/dense_128key.cu, fast-path blocks only).  Usage: BLEND_LIB=...libblend_tp.so
python scripts/trace_phases.py c4"""
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
t = t[t[:, 45] > 0]
n = t[:, 45:46]
names = ["s_full wait", "S ld + mask", "exp / sum / pack", "P st issue", "st wait+fence+arrive"]
per = t[:, 40:45] / n
print(f"{w.name}: {len(t)} CTAs, {np.median(n):.0f} fast blocks each; cycles per block (median over CTAs)")
for i, nm in enumerate(names):
    print(f"  {nm:22s} {np.median(per[:, i]):8.1f}")
print(f"  {'total':22s} {np.median(per.sum(1)):8.1f}")
ghz = (t[:, 49] - t[:, 48]) / (t[:, 6] - t[:, 0])
print(f"  SM clock over the kernel (clock64 / globaltimer): {np.median(ghz):.3f} GHz; "
      f"kernel {np.median(t[:, 6] - t[:, 0]) / 1e3:.1f} us; blocks of unit 0 per CTA {np.median(n):.0f}")
