"""Pins the CPU oracle (oracle/fq_oracle.c) before it is trusted as the checker:
(1) the reference's own known answers (tests/golden/kat.json, cited file:line),
(2) golden fixtures produced by the unmodified reference (tests/golden/*.npz,
    tests/golden/make_golden.py), and
(3) the unmodified reference built here (oracle/_ref), live, on random layers.
"""
import glob
import json
import os

import numpy as np
import pytest

from oracle import InvalidArgument, ReferenceRuntimeError

GOLDEN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")
KAT = json.load(open(os.path.join(GOLDEN, "kat.json")))
FIXTURES = sorted(glob.glob(os.path.join(GOLDEN, "*.npz")))


def kat_maxes(p):
    if "maxes" in p:
        return np.array(p["maxes"], np.float64)
    spec = p["maxes_spec"]
    m = np.full(spec["n"], spec["value"])
    m[: spec["head"]] = spec["head_value"]
    return m


@pytest.mark.parametrize("p", KAT["plans"], ids=lambda p: p["cite"])
def test_plan_known_answers(port, p):
    e, off, c, padded = port.build_plan(kat_maxes(p), p["t"])
    assert c == p["c_extend"] and padded == p["padded"]
    if "ext" in p:
        assert list(e) == p["ext"]
    if "slots0" in p:
        k = len(e)
        assert [0] + [k + int(off[0]) + q for q in range(int(e[0]))] == p["slots0"]


@pytest.mark.parametrize("p", KAT["invalid_plans"], ids=lambda p: p["cite"])
def test_plan_validation(port, p):
    with pytest.raises(InvalidArgument):
        port.build_plan(np.array(p["maxes"], np.float64), p["t"])


@pytest.mark.parametrize("p", KAT["splits"], ids=lambda p: p["cite"] + f" x={p['x']}")
def test_split_known_answers(port, p):
    e, _, _, _ = port.build_plan(np.array(p["plan_maxes"]), p["t"])
    flat, sat = port.flatten_columns(np.array([[p["x"]]]), p["t"], e)
    slots = [0] + [1 + q for q in range(int(e[0]))]
    got = [flat[0, s] for s in slots][: len(p["slots"])]
    assert got == p["slots"] and sat == p["saturated"]
    assert not flat[0, len(slots):].any()


@pytest.mark.parametrize("p", KAT["strict_overflow"], ids=lambda p: p["cite"])
def test_strict_flatten_overflow(port, p):
    e, _, _, _ = port.build_plan(np.array(p["plan_maxes"]), p["t"])
    with pytest.raises(ReferenceRuntimeError):
        port.flatten_columns(np.array([[p["x"]]]), p["t"], e, strict=True)


@pytest.mark.parametrize("p", KAT["repeat"], ids=lambda p: p["cite"])
def test_repeat_known_answers(port, p):
    e, _, _, padded = port.build_plan(np.array(p["plan_maxes"]), p["t"])
    rep = port.repeat_channels(np.array([[p["w"]]]), e)
    assert rep.shape == (padded, 1)
    assert list(rep[: len(p["rows"]), 0]) == p["rows"] and not rep[len(p["rows"]):].any()
    rc = port.repeat_columns(np.array([[p["w"]]]), e)
    assert list(rc[0, : len(p["rows"])]) == p["rows"] and not rc[0, len(p["rows"]):].any()


@pytest.mark.parametrize("p", KAT["quantize"], ids=lambda p: p["cite"])
def test_quantize_known_answers(port, p):
    q, s = port.quantize(np.array(p["m"]), p["bits"], p["scale"])
    assert list(q) == p["q"]
    assert s == pytest.approx(p["scale_out"], rel=1e-15)


@pytest.mark.parametrize("p", KAT["degenerate_quantize"], ids=lambda p: p["cite"])
def test_degenerate_scale(port, p):
    with pytest.raises(ReferenceRuntimeError):
        port.quantize(np.array(p["m"]), p["bits"])


@pytest.mark.parametrize("p", KAT["accumulator_bound"], ids=lambda p: str(p["inner"]))
def test_accumulator_bound(port, p):
    assert bool(port.lib.fqo_accumulator_bound_ok(p["qx"], p["qw"], p["inner"])) == p["ok"]


def test_flatten_pair_product(port):
    p = KAT["flatten_pair"][0]
    ex, _, _, _ = port.build_plan(np.array([p["x"]]), p["t_x"])
    assert list(ex) == p["ext_x"]
    x1, _ = port.flatten_columns(np.array([[p["x"]]]), p["t_x"], ex, strict=True)
    w1 = port.repeat_channels(np.array([[p["w"]]]), ex)
    ew, _, _, _ = port.build_plan(np.abs(w1).max(axis=1), p["t_w"])
    wf = port.flatten_rows(w1, p["t_w"], ew)
    xf = port.repeat_columns(x1, ew)
    assert float((xf @ wf)[0, 0]) == pytest.approx(p["product"], abs=1e-12)


@pytest.mark.parametrize("path", FIXTURES, ids=os.path.basename)
def test_oracle_reproduces_reference_fixtures(port, path):
    g = np.load(path)
    bits = int(g["bits"])
    L = port.quantize_layer(g["weight"], g["calib"], bits)
    assert L.t_x == float(g["t_x"]) and L.t_w == float(g["t_w"])
    assert np.array_equal(L.s, g["s"]) and np.array_equal(L.e_x, g["e_x"])
    assert np.array_equal(L.e_w, g["e_w"]) and np.array_equal(L.wq, g["wq"].astype(np.int32))
    assert L.s_w == float(g["s_w"]) and L.act_scale == float(g["act_scale"])
    for tag in ("", "_sat"):
        x = g["x"] * (3.0 if tag else 1.0)
        y, sat, qx, acc = port.run_layer(L, x, debug=True)
        assert sat == int(g["sat" + tag])
        assert np.array_equal(qx, g["qx" + tag].astype(np.int32))
        assert np.array_equal(acc, g["acc" + tag].astype(np.int64))
        assert np.array_equal(y, g["y" + tag])


@pytest.mark.parametrize("seed", range(6))
def test_oracle_vs_live_reference(port, ref, seed):
    rng = np.random.default_rng(seed)
    k = int(rng.choice([64, 96, 160, 256]))
    n = int(rng.choice([32, 80, 128]))
    w, calib, x, _ = ref.synthetic_layer(seed + 10, in_channels=k, out_channels=n, rows=16,
                                         samples=3, outlier_min=float(rng.uniform(5, 30)),
                                         outlier_max=float(rng.uniform(40, 120)))
    mode = 1 if seed % 2 == 0 else 2
    rl = ref.quantize_layer(w, calib, mode=mode, gamma=1.86 if mode == 1 else 1e6,
                            beta=float(rng.uniform(1.0, 1.6)))
    L = rl.to_layer()
    # the C restatement of quantize_layer (bits pinned to the reference's choice)
    beta = float(rng.uniform(1.0, 1.6))
    rl = ref.quantize_layer(w, calib, mode=mode, gamma=1.86 if mode == 1 else 1e6, beta=beta)
    L = rl.to_layer()
    P = port.quantize_layer(w, calib, L.bits, beta=beta)
    assert (P.t_x, P.t_w, P.s_w, P.act_scale) == (L.t_x, L.t_w, L.s_w, L.act_scale)
    assert np.array_equal(P.wq, L.wq) and np.array_equal(P.e_w, L.e_w)
    # run_layer on the reference recipe, including saturating inputs
    for scale in (1.0, 2.5):
        xs = x * scale
        y_ref, s_ref = rl.run_layer(xs)
        y, s, qx, _ = port.run_layer(L, xs, debug=True)
        q_ref, _ = rl.quantized_acts(xs)
        assert np.array_equal(qx, q_ref) and s == s_ref and np.array_equal(y, y_ref)


def test_int_matmul_vs_reference(port, ref):
    rng = np.random.default_rng(7)
    for _ in range(10):
        m, kk, n = rng.integers(1, 40, 3)
        bx, bw = rng.choice([4, 8], 2)
        qx = rng.integers(-((1 << (bx - 1)) - 1), 1 << (bx - 1), (m, kk)).astype(np.int32)
        qw = rng.integers(-((1 << (bw - 1)) - 1), 1 << (bw - 1), (kk, n)).astype(np.int32)
        a = port.int_matmul_raw(qx, qw, int(bx), int(bw))
        assert np.array_equal(a, ref.int_matmul_raw(qx, qw, int(bx), int(bw)))
        assert np.array_equal(a, qx.astype(np.int64) @ qw.astype(np.int64))


def test_calibration_stages_vs_reference(port, ref):
    rng = np.random.default_rng(3)
    calib = rng.standard_normal((3, 20, 50)) * rng.uniform(0.1, 30, 50)
    m = ref.collect_channel_maxes(calib)
    for clip in (True, False):
        assert port.derive_truncation(m, 1.3, clip) == ref.derive_truncation(m, 1.3, clip)
    wm = np.abs(rng.standard_normal((50, 30))).max(axis=1)
    assert np.array_equal(port.smoothing_scales(m, wm, 0.5), ref.smoothing_scales(m, wm, 0.5))
