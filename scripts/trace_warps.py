import ctypes as C, sys, numpy as np, torch
sys.path.insert(0, ".")
import bench, paper_2411_16102_b200 as B
from harness.run import device_batch
w = bench.make_workload(sys.argv[1])
db = device_batch(w, tree_kw=dict(num_sms=148))
for _ in range(3): db.run()
torch.cuda.synchronize()
tr = torch.zeros((297, 64), dtype=torch.int64, device="cuda")
L = B.lib(); L.blend_internal_set_trace.argtypes = [C.c_void_p]
L.blend_internal_set_trace(tr.data_ptr()); db.run(flags=B.SERIALIZE); torch.cuda.synchronize(); L.blend_internal_set_trace(None)
t = tr.cpu().numpy()[:148].astype(np.float64)
ok = t[:, 24] > 0
t = t[ok]
for j in range(4):
    blk = t[:, 24 + 8 * j: 32 + 8 * j]
    rel = (blk - blk.min(axis=1, keepdims=True)) / 1e3   # us after the earliest warp of this block
    print(f"block {20 + j}: median lag per softmax warp (us) A:", np.round(np.median(rel[:, :4], axis=0), 3), " B:", np.round(np.median(rel[:, 4:], axis=0), 3))
