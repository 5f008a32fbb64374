"""C4 grid density sweep (BASELINE configs[3] "compute density t sweep,
prefix sharing ratio 0.5"; PAPER P:28 grid): the stored counts
(synth/c4_counts.json, written by scripts/solve_c4_counts.py) give, on the realised
samples, a root density within 2 % of t and a sharing ratio within 0.02 of 0.5, both
computed by the oracle (B200 constants of SURVEY §8)."""
import pytest

from oracle import tree as T
from synth import workloads as W

COMPUTE, BW, KVB = 1391.8e12, 6537e9, 1024 * 32 * 4


@pytest.mark.parametrize("t", W.C4_T)
def test_c4_realised_density_and_sharing(t):
    w = W.c4_grid(t=t)
    assert w.n_req == 40000 and sum(W.c4_counts(t)) == 40000
    v = T.build(w)
    rho = T.density(*T.root_key(v), COMPUTE, BW, KVB)
    s = T.sharing_ratio(w, v)
    assert abs(rho / t - 1) <= 0.02, (t, rho)
    assert abs(s - 0.5) <= 0.02, (t, s)


def test_c4_density_ordering():
    # more OpenVid decodes (memory-heavy, d ~ 16K) -> lower density
    nv = [W.c4_counts(t)[1] for t in W.C4_T]
    assert nv == sorted(nv, reverse=True)
