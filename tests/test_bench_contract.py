"""The committed bench lines (profiles/<latest>/) carry every key of the driver's bench
contract, with consistent values (CPU only: reads JSON, runs nothing)."""
import json
import os

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
LATEST = os.path.join(ROOT, "profiles", "r1h")


def _load(name):
    p = os.path.join(LATEST, name)
    if not os.path.exists(p):
        pytest.skip(f"{p} not committed")
    return json.load(open(p))


def test_default_line_keys():
    d = _load("bench_c2_default.json")
    for k in ("metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step", "higher_is_better",
              "scaling", "vs_baseline", "dtype", "data", "config", "roofline", "cpu_baseline", "e2e",
              "clocks", "gpu_launches"):
        assert k in d, k
    assert d["n_gpus"] == 1 and d["warmup"] >= 3 and d["higher_is_better"] is True
    assert d["config"]["workload"] == "c2_mmlu_decode"
    r = d["roofline"]
    assert r["bound"] in ("hbm", "tensor", "alu") and r["unit"] in ("GB/s", "TFLOP/s")
    assert r["frac"] == pytest.approx(r["achieved"] / r["peak"], rel=1e-6)
    assert r["traffic"] is None or r["traffic"] > 0
    c = d["cpu_baseline"]
    assert c["kind"] == "oracle" and c["cores"] >= 1 and c["value"] > 0 and c["sample"]
    e = d["e2e"]
    assert e["h2d_bytes_per_step"] > 0 and e["d2h_bytes_per_step"] > 0 and e["value"] != d["value"]
    assert d["gpu_launches"] > 0
    assert not set(d["clocks"]["reasons"]) & {"hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown"}
    # tokens/s = query tokens per step / step time
    assert d["value"] == pytest.approx(d["plan"]["n_tokens"] / (d["ms_per_step"] * 1e-3), rel=1e-3)


def test_reference_line_keys():
    d = _load("bench_reference.json")
    assert d["impl"] == "reference"
    assert d["cpu_baseline"]["value"] == d["value"]
    assert d["e2e"]["h2d_bytes_per_step"] == 0 and d["e2e"]["d2h_bytes_per_step"] == 0
