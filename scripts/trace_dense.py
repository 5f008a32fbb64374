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
if not np.all(np.isnan(rel[:, 20])) and np.nanmax(rel[:, 20:60]) > 0:
    # BLEND_TRACE_UNITS: slots 20+4k.. = start, first S, last P, epilogue end of the k-th
    # unit of a CTA (tile A); the unit's 64-key block count comes from the plan image
    sys.path.insert(0, "tests")
    from plan_sim import plan_image  # noqa: E402
    du = plan_image(db.tree)["dunits"]
    G = int(used.sum())
    epb = 64 // min(w.page_size, 64)
    print("per-unit (BLEND_TRACE_UNITS), medians over CTAs [us]: start->S0, S0->lastP, lastP->end, "
          "end->next start, 64-key blocks, us per block")
    tot_b = tot_t = 0.0
    for k in range(10):
        a, s0, lp, en = (rel[:, 20 + 4 * k + i] for i in range(4))
        nxt = rel[:, 20 + 4 * (k + 1)] if k < 9 else np.full_like(a, np.nan)
        ui = np.array([k * G + ((G - 1 - b) if k & 1 else b) for b in range(G)])
        uc = np.minimum(ui, len(du) - 1)
        nb = np.where(ui < len(du), (du[uc, 5] - du[uc, 4] + epb - 1) // epb, 0)
        per = (lp - s0) / np.maximum(nb - 1, 1)
        print(f"  unit {k}: {np.nanmedian(s0 - a):6.2f} {np.nanmedian(lp - s0):7.2f} {np.nanmedian(en - lp):6.2f} "
              f"{np.nanmedian(nxt - en) if k < 9 else float('nan'):6.2f}   {np.median(nb):5.1f}  {np.nanmedian(per):5.3f}")
        if k < 9:
            tot_t += np.nansum(nxt - a)
            tot_b += float(nb.sum())
    print(f"  mean unit-to-unit time per 64-key block: {tot_t / max(tot_b, 1):.3f} us")
for k in list(range(7)) + [60, 62, 63, 61] + list(range(8, 20)):
    col = rel[:, k]
    if np.all(np.isnan(col)):
        continue
    nm = names.get(k, f"S{(k - 8) // 2}" if k % 2 == 0 else f"P{(k - 8) // 2}")
    print(f"{nm:>6}: median {np.nanmedian(col):8.2f} us  min {np.nanmin(col):8.2f}  max {np.nanmax(col):8.2f}")
if tall[:148, 45].max() > 0:
    # BLEND_TRACE_UNITS: clock64 sums over ALL units of tile A per CTA (slots 40..45)
    a = tall[:148, 40:46].astype(np.float64)
    keep = a[:, 5] > 0
    a = a[a[:, 5] > 0]
    units, blocks = a[:, 5], a[:, 4]
    tot = a[:, 0:4].sum(1)
    print(f"all units (tile A, clock64; median over CTAs): {np.median(units):.0f} units, {np.median(blocks):.0f} "
          "64-key blocks per CTA")
    for i, nm in enumerate(["start -> first S", "first S -> last P", "last P -> epilogue end", "epilogue end -> next start"]):
        print(f"  {nm:28s} {np.median(a[:, i] / units):9.0f} cycles / unit  ({np.median(a[:, i] / tot) * 100:5.1f} %)")
    print(f"  blocks: {np.median(a[:, 1] / np.maximum(blocks - units, 1)):.0f} cycles per block after the first")
    b = tall[:148, 46:48].astype(np.float64)[tall[:148, 45] > 0]
    if b[:, 1].sum() > 0:
        two_c, two_b = a[:, 1] - b[:, 0], blocks - b[:, 1]
        print(f"  single-tile units: {np.median(b[:, 1]):.0f} blocks per CTA at {np.median(b[:, 0] / np.maximum(b[:, 1], 1)):.0f} "
              f"cycles per block; two-tile units: {np.median(two_b):.0f} blocks at {np.median(two_c / np.maximum(two_b, 1)):.0f}")
if tall[:148, 56].max() > 0:
    ph = tall[:148, 48:58].astype(np.float64)
    ph = ph[ph[:, 8] > 0]
    print("softmax phases per fast block (tile A, clock64 cycles, median over CTAs): S wait, S ld, exps, P st + arrive")
    for nm, o, c in (("two-tile units", 0, 8), ("single-tile units", 4, 9)):
        n = np.maximum(ph[:, c], 1)
        print(f"  {nm:18s} " + "  ".join(f"{np.median(ph[:, o + i] / n):7.0f}" for i in range(4)))
