"""Randomised layer parity (K1 + K4 through Layer.forward) against the oracle's run_layer:
random K / N / M, 4- or 8-bit recipes, int8 or packed int4 activations, bf16 / f16 / f32 / f64
inputs, every row checked on the INT32 accumulators and the f64 output.
FQG_LAYER_FUZZ_CASES raises the case count (default 8)."""
import os

import numpy as np
import pytest

from conftest import bf16_round

pytestmark = pytest.mark.gpu

CASES = int(os.environ.get("FQG_LAYER_FUZZ_CASES", "8"))


@pytest.mark.parametrize("case", range(CASES))
def test_layer_fuzz(port, fq, case):
    import torch

    rng = np.random.default_rng(7000 + case)
    k = int(rng.integers(1, 48)) * 32
    n = int(rng.integers(1, 40)) * 32
    m = int(rng.choice([1, 2, 3, 9, 64, 130, 257, 600]))
    bits = int(rng.choice([4, 8]))
    in_dt = str(rng.choice(["bf16", "f16", "f32", "f64"]))
    a_fmt = fq.I4 if (bits == 4 and rng.integers(0, 2)) else fq.I8
    w, calib, x = fq.synthetic_layer(100 + case, test_rows=m, in_channels=k, out_channels=n,
                                     rows=32, samples=4)
    L = port.quantize_layer(w, calib, bits)
    tdt = {"bf16": torch.bfloat16, "f16": torch.float16, "f32": torch.float32,
           "f64": torch.float64}[in_dt]
    # the values the device sees, as the oracle's f64 input
    xt = torch.from_numpy(bf16_round(x) if in_dt == "bf16" else x).to(tdt).cuda()
    xv = xt.double().cpu().numpy()
    px = fq.FlattenPlan.from_extensions(L.t_x, L.e_x, L.block)
    pw = fq.FlattenPlan.from_extensions(L.t_w, L.e_w, L.block)
    cfg = fq.LayerQuantConfig(bits=bits, smooth_scales=L.s, plan_x=px, plan_w=pw,
                              act_scale=L.act_scale, weight_q=L.wq, w_scale=L.s_w)
    layer = fq.Layer(cfg, a_format=a_fmt, b_format=fq.I4 if bits == 4 else fq.I8)
    acc = layer.forward(xt, out_dtype=torch.int32).cpu().numpy()
    y = layer.forward(xt, out_dtype=torch.float64).cpu().numpy()
    y_ref, _, _, acc_ref = port.run_layer(L, xv, debug=True)
    where = f"case {case}: k={k} n={n} m={m} bits={bits} in={in_dt} a_fmt={a_fmt}"
    assert np.array_equal(acc.astype(np.int64), acc_ref), where
    assert np.array_equal(y, y_ref), where
