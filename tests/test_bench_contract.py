"""The bench.py JSON contract, checked on the committed evidence lines (profiles/*_bench.jsonl):
every key the driver and the judge read is present with the right shape."""
import glob
import json
import os

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def latest_bench_lines():
    files = sorted(glob.glob(os.path.join(ROOT, "profiles", "r*_bench.jsonl")))
    assert files, "no committed bench evidence under profiles/"
    with open(files[-1]) as f:
        return [json.loads(line) for line in f if line.strip().startswith("{")]


def test_main_line_keys():
    main = next(d for d in latest_bench_lines() if d.get("impl") != "reference" and "subresults" in d)
    for key in ("metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step",
                "higher_is_better", "scaling", "vs_baseline", "dtype", "data", "config",
                "roofline", "cpu_baseline", "e2e", "gpu_launches", "clocks"):
        assert key in main, key
    assert main["warmup"] >= 3
    assert main["config"]["workload"] and "l2" in main["config"]
    r = main["roofline"]
    for key in ("bound", "achieved", "peak", "unit", "frac", "traffic"):
        assert key in r, key
    assert r["bound"] in ("hbm", "tensor") and 0 < r["frac"] < 1
    assert abs(r["achieved"] / r["peak"] - r["frac"]) < 1e-9
    c = main["cpu_baseline"]
    for key in ("value", "unit", "cores", "kind", "sample"):
        assert key in c, key
    assert c["kind"] in ("reference", "port")
    e = main["e2e"]
    for key in ("value", "unit", "h2d_bytes_per_step", "d2h_bytes_per_step"):
        assert key in e, key
    assert e["h2d_bytes_per_step"] > 0 and e["d2h_bytes_per_step"] > 0
    assert main["gpu_launches"] > 0
    for key in ("sm_mhz", "sm_max_mhz", "reasons"):
        assert key in main["clocks"], key


def test_reference_arm_line():
    ref = [d for d in latest_bench_lines() if d.get("impl") == "reference"]
    if not ref:
        pytest.skip("no reference-arm line in the latest evidence")
    d = ref[0]
    assert "unavailable" in d or ("value" in d and d["e2e"]["h2d_bytes_per_step"] == 0)
    if "value" in d:
        assert d["cpu_baseline"]["kind"] in ("reference", "port")
