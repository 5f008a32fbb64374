"""Input generator checks (synth/ is input generation only)."""
import numpy as np
import torch

from synth import values as V
from synth import workloads as W


def test_splitmix64_known_values():
    # splitmix64 (Vigna) with state 0 / 1: first outputs are the published constants
    assert int(V.mix(np.array([0], np.uint64))[0]) == 0xE220A8397B1DCDAF
    assert int(V.mix(np.array([1], np.uint64))[0]) == 0x910A2DEC89025CC1


def test_grid_values_exact_in_bf16():
    z = np.arange(256, dtype=np.uint64) << np.uint64(56)
    g = V.grid(z)
    assert g.min() == -1.0 and g.max() == 127 / 128
    t = torch.tensor(g, dtype=torch.float64)
    assert torch.equal(t.to(torch.bfloat16).to(torch.float64), t)
    t8 = 8 * t
    assert torch.equal(t8.to(torch.bfloat16).to(torch.float64), t8)


def test_kv_depends_only_on_prefix():
    a = np.array([5, 6, 7, 8, 9], np.int32)
    b = np.array([5, 6, 7, 1, 2, 3], np.int32)
    Ka, Va = V.path_kv(a, 11, 2, 64)
    Kb, Vb = V.path_kv(b, 11, 2, 64)
    assert np.array_equal(Ka[:3], Kb[:3]) and np.array_equal(Va[:3], Vb[:3])
    assert not np.array_equal(Ka[3], Kb[3])
    assert not np.array_equal(Ka, Va[:, :, :])


def test_q_depends_on_global_id():
    q0 = V.q_values(0, np.arange(2), 3, 4, 64)
    q1 = V.q_values(1, np.arange(2), 3, 4, 64)
    assert not np.array_equal(q0, q1)
    assert np.array_equal(V.q_values(7, np.array([1]), 3, 4, 64)[0], V.q_values(7, np.arange(2), 3, 4, 64)[1])


def test_workload_shapes():
    w = W.c3_burst_openvid()
    assert w.n_req == 1024 and w.sum_q == 64 * 512 + 960
    w = W.c2_mmlu_decode()
    assert w.n_req == 256 and np.all(w.q_len == 1)
    assert np.all(np.diff(w.tok_off) >= 1024 + 80)
    w = W.c1_tiny("c")
    assert w.n_req == 9 and int(w.q_len[8]) == 64
