import sys, numpy as np, torch
sys.path.insert(0, '.')
import paper_2411_16102_b200 as B
from harness.run import device_batch
from oracle import attention as A
from tests.helpers import random_workload
seed = 5
hq, hkv = [(8, 2), (32, 8), (16, 1), (4, 4)][seed % 4]
w = random_workload(seed, hq=hq, hkv=hkv, d=128 if seed % 2 else 64, kv_dtype="bf16",
                    page_size=[16, 32, 64, 128][seed % 4], max_seg=300, n_req=int(8 + seed * 5))
ref = A.attention_workload(w)
qo = np.concatenate([[0], np.cumsum(w.q_len)])
for kw in (dict(), dict(force_class=1, min_sep_len=0), dict(rows_min=16, min_sep_len=0)):
    db = device_batch(w, tree_kw=kw)
    for path in (B.PATH_AUTO, B.PATH_GENERIC, B.PATH_NO_TCGEN05):
        for flags in (0, 1):
            db.out.zero_(); db.run(path=path, flags=flags); torch.cuda.synchronize()
            out = db.out.float().cpu().numpy()
            worst = max((float(np.abs(out[qo[r]:qo[r+1]] - ref[r][0]).max()), r) for r in range(w.n_req))
            print(kw, 'path', path, 'flags', flags, 'worst', worst, 'info', db.info['n_dense_units'], db.info['n_stream_units'])
