"""Host-side product logic (no GPU): plan arithmetic, the composite gather maps,
the offline recipe builder and the synthetic generator of libfqg.so, checked
against the reference known answers, the golden fixtures and the oracle."""
import glob
import json
import os

import numpy as np
import pytest

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
def test_build_flatten_plan_known_answers(fq, p):
    plan = fq.build_flatten_plan(kat_maxes(p), p["t"])
    assert plan.c_extend == p["c_extend"] and plan.padded_width == p["padded"]
    if "ext" in p:
        assert list(plan.extensions) == p["ext"]
    if "slots0" in p:
        assert plan.slot_of(0) == p["slots0"]


@pytest.mark.parametrize("p", KAT["invalid_plans"], ids=lambda p: p["cite"])
def test_build_flatten_plan_validation(fq, p):
    with pytest.raises(fq.FqgInvalidArgument):
        fq.build_flatten_plan(np.array(p["maxes"], np.float64), p["t"])


@pytest.mark.parametrize("p", KAT["splits"], ids=lambda p: p["cite"] + f" x={p['x']}")
def test_split_against_threshold(fq, port, p):
    for a in (abs(p["x"]), 7.0, 6.0, 6.5, 0.0, 1e-300):
        assert fq.split_against_threshold(a, p["t"]) == port.split(a, p["t"])


def test_split_random_vs_oracle(fq, port):
    rng = np.random.default_rng(5)
    for _ in range(2000):
        t = float(rng.uniform(0.01, 50))
        a = float(abs(rng.standard_normal()) * t * rng.integers(1, 60))
        assert fq.split_against_threshold(a, t) == port.split(a, t)


def test_plans_random_vs_oracle(fq, port):
    rng = np.random.default_rng(9)
    for _ in range(50):
        k = int(rng.integers(1, 300))
        m = np.abs(rng.standard_normal(k)) * rng.uniform(0.1, 40, k)
        t = float(rng.uniform(0.2, 5))
        block = int(rng.choice([1, 8, 32, 128]))
        plan = fq.build_flatten_plan(m, t, block)
        e, off, c, padded = port.build_plan(m, t, block)
        assert np.array_equal(plan.extensions, e[:k]) and np.array_equal(plan.ext_offset, off[:k])
        assert (plan.c_extend, plan.padded_width) == (c, padded)


def _oracle_maps(port, e_x, e_w, block=32):
    """Independent construction of the composite maps from the oracle's own
    repeat_columns / repeat_channels on index rows (flatten.cpp:136-174)."""
    k = len(e_x)
    c1 = port.repeat_columns(np.zeros((1, k)), e_x).shape[1]
    # flat column r -> source channel j (+1; 0 for padding)
    src = port.repeat_columns((np.arange(k) + 1.0)[None, :], e_x, block)[0].astype(np.int64)
    # final column k' -> flat column r (+1; 0 for padding)
    fcol = port.repeat_columns((np.arange(c1) + 1.0)[None, :], e_w, block)[0].astype(np.int64)
    off = np.concatenate([[0], np.cumsum(e_x)[:-1]])
    offw = np.concatenate([[0], np.cumsum(e_w)[:-1]])
    kp = len(fcol)
    amap = np.full(kp, -1, np.int64)
    wmap = np.full(kp, -1, np.int64)
    wcap = np.ones(kp, np.int64)
    for kq in range(kp):
        r = fcol[kq] - 1
        if r < 0 or src[r] == 0:
            continue
        j = src[r] - 1
        p_x = 0 if r < k else r - k - off[j] + 1
        amap[kq] = (j << 12) | p_x
        p_w = 0 if kq < c1 else kq - c1 - offw[r] + 1
        wmap[kq] = (j << 12) | p_w
        wcap[kq] = e_w[r] + 1
    return amap, wmap, wcap


@pytest.mark.parametrize("path", FIXTURES[:3], ids=os.path.basename)
def test_gather_maps_vs_oracle(fq, port, path):
    import ctypes as C

    g = np.load(path)
    e_x = np.ascontiguousarray(g["e_x"], np.int64)
    e_w = np.ascontiguousarray(g["e_w"], np.int64)
    cap = 4 * (len(e_x) + int(e_x.sum()) + int(e_w.sum())) + 256
    amap = np.zeros(cap, np.int32)
    wmap = np.zeros(cap, np.int32)
    wcap = np.zeros(cap, np.int32)
    kp = C.c_int64()
    fq.check(fq.lib().fqg_gather_maps(e_x.ctypes.data, len(e_x), 32, e_w.ctypes.data, 32,
                                      amap.ctypes.data, wmap.ctypes.data, wcap.ctypes.data,
                                      C.byref(kp), cap))
    ra, rw, rc = _oracle_maps(port, e_x, e_w)
    n = kp.value
    assert n == len(ra)
    assert np.array_equal(amap[:n], ra) and np.array_equal(wmap[:n], rw)
    pad = rw < 0
    assert np.array_equal(wcap[:n][~pad], rc[~pad])


@pytest.mark.parametrize("path", FIXTURES, ids=os.path.basename)
def test_synthetic_generator_reproduces_reference(fq, path):
    """The product generator is bit-identical to fq::make_synthetic_layer."""
    g = np.load(path)
    name = os.path.basename(path)
    index = {"ref128_o1": 0, "ref128_o2": 1, "k256_n96_o1": 2, "k192_n160_o2": 3}[name[:-4]]
    s, r, k = g["calib"].shape
    n = g["weight"].shape[1]
    w, calib, x = fq.synthetic_layer(index, in_channels=k, out_channels=n, rows=r, samples=s)
    assert np.array_equal(w, g["weight"]) and np.array_equal(calib, g["calib"])
    assert np.array_equal(x, g["x"])


@pytest.mark.parametrize("path", FIXTURES, ids=os.path.basename)
def test_recipe_builder_reproduces_reference(fq, path):
    """quantize_layer's host stages (smoothing, truncation, both plans, s_x)."""
    g = np.load(path)
    cfg = fq.quantize_layer(g["weight"], g["calib"], int(g["bits"]))
    assert np.array_equal(cfg.smooth_scales, g["s"])
    assert cfg.plan_x.threshold == float(g["t_x"]) and cfg.plan_w.threshold == float(g["t_w"])
    assert np.array_equal(cfg.plan_x.extensions, g["e_x"])
    assert np.array_equal(cfg.plan_w.extensions, g["e_w"])
    assert cfg.act_scale == float(g["act_scale"])


def test_recipe_builder_ablations_vs_oracle(fq, port):
    rng = np.random.default_rng(2)
    w = rng.standard_normal((96, 40))
    calib = rng.standard_normal((2, 12, 96)) * rng.uniform(0.2, 25, 96)
    for smooth in (True, False):
        for clip in (True, False):
            cfg = fq.quantize_layer(w, calib, 8, smooth=smooth, clip=clip, beta=1.1)
            L = port.quantize_layer(w, calib, 8, smooth=smooth, clip=clip, beta=1.1)
            assert cfg.plan_x.threshold == L.t_x and cfg.plan_w.threshold == L.t_w
            assert np.array_equal(cfg.plan_w.extensions, L.e_w)


def test_collect_channel_maxes(fq, port):
    rng = np.random.default_rng(4)
    calib = rng.standard_normal((3, 17, 33))
    m = fq.collect_channel_maxes(calib)
    assert np.array_equal(m, np.abs(calib).max(axis=(0, 1)))


def test_layer_creation_fails_loudly_without_gpu(fq):
    """No CPU fallback: creating a device layer without a CUDA device raises."""
    import torch

    if torch.cuda.is_available():
        pytest.skip("GPU present")
    plan = fq.FlattenPlan.from_extensions(1.0, np.zeros(8, np.int64))
    planw = fq.FlattenPlan.from_extensions(1.0, np.zeros(32, np.int64))
    cfg = fq.LayerQuantConfig(bits=8, smooth_scales=np.ones(8), plan_x=plan, plan_w=planw,
                              act_scale=1.0 / 127, weight_q=np.ones((32, 4), np.int32),
                              w_scale=0.1)
    with pytest.raises(fq.FqgError) as ei:
        fq.Layer(cfg)
    assert ei.value.code == -4  # FQG_ERR_CUDA
