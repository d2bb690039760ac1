"""GPU parity of the K4 epilogue on every kernel path: output dtype x bias dtype.

Semantics (quantize.cpp:190-198 + the north_star bias): y = RN_out(RN64(RN64(
double(acc) * RN64(s_x * s_w)) + double(bias[n]))): the reference's f64 output,
plus the bias in f64, rounded once to the output type. Bias is a build
extension (the reference has none); with a zero bias the result is the
reference output exactly.

Paths (asserted with fqg_gemm_plan, so a dispatch change cannot silently skip
one): the 1-CTA 128 x N kernel, the CTA-pair kernel with 256 x 256 tiles, the
pair kernel with 256 x 512 tiles, the 512 x 256 tiles of packed int4 weights,
the CUDA-core path for decode-size M (1-2 rows, int8 weights), and split-K with its in-kernel fix-up (including the orphaned-chunk path a split
takes when its peers are not resident, forced by debug bit 128).
"""
import ctypes as C
import os
import subprocess
import sys

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

PATHS = {  # name: (M, N, K', expected plan {kernel, tile_n, splits>1})
    "one_cta": (100, 128, 512, (1, None, False)),
    "pair_small_m_splitk": (100, 2048, 2048, (2, 256, True)),
    "pair_256x256": (1024, 2560, 512, (2, 256, False)),
    "pair_256x512": (2048, 3072, 256, (2, 512, False)),
    "splitk_fixup_ragged": (200, 1000, 2048, (2, 256, True)),
    "pair_512x256_int4_weights": (2048, 3072, 256, (2, 256, False)),  # packed B: 512-row tiles
    "gemv_decode": (2, 1000, 2048, (3, None, False)),  # M <= 2: CUDA-core weight stream
    "gemv_decode_one_row": (1, 4100, 1024, (3, None, False)),
}
PACKED_B = {"pair_512x256_int4_weights"}
OUTS = ["f16", "bf16", "f32", "f64"]
BIASES = [None, "f64", "f32", "f16", "bf16"]


def _rn_bf16(v):
    mant, ex = np.frexp(v)
    return np.ldexp(np.round(mant * 256.0), ex - 8)


def _round_out(v, out):
    if out == "f16":
        return v.astype(np.float16).astype(np.float64)
    if out == "bf16":
        return _rn_bf16(v)
    if out == "f32":
        return v.astype(np.float32).astype(np.float64)
    return v


def plan(fq, m, n, kp, a_fmt, b_fmt, y_dtype):
    from paper_2402_17985_b200 import _lib

    info = _lib.GemmPlan()
    fq.check(fq.lib().fqg_gemm_plan(m, n, kp, a_fmt, b_fmt, y_dtype, C.byref(info)))
    return info


@pytest.mark.parametrize("path", sorted(PATHS))
def test_epilogue_out_and_bias(fq, path):
    import torch

    from paper_2402_17985_b200 import _lib

    m, n, kp, (kern, tile_n, split) = PATHS[path]
    g = torch.Generator().manual_seed(m * 7 + n)
    a = torch.randint(-127, 128, (m, kp), dtype=torch.int8, generator=g)
    packed = path in PACKED_B
    b = torch.randint(-7 if packed else -127, 8 if packed else 128, (n, kp), dtype=torch.int8,
                      generator=g)
    acc = a.numpy().astype(np.int64) @ b.numpy().astype(np.int64).T
    if packed:  # FQG_I4: per group of 32 k, byte i = q[i] & 15 | q[16 + i] << 4
        nib = (b.numpy().astype(np.int32) & 15).reshape(n, kp // 32, 2, 16)
        b = torch.from_numpy((nib[:, :, 0, :] | (nib[:, :, 1, :] << 4)).astype(np.uint8)
                             .reshape(n, kp // 2).view(np.int8))
    b_code, ldb = (_lib.I4, kp // 2) if packed else (_lib.I8, kp)
    sx, sw = 3.7e-5, 0.0123
    s = sx * sw  # quantize.cpp:193, formed once in f64
    scale = torch.tensor([sx, sw], dtype=torch.float64, device="cuda")
    ad, bd = a.cuda(), b.cuda()
    tdt = {"f16": torch.float16, "bf16": torch.bfloat16, "f32": torch.float32,
           "f64": torch.float64}
    code = {"f16": _lib.F16, "bf16": _lib.BF16, "f32": _lib.F32, "f64": _lib.F64}
    st = torch.cuda.current_stream().cuda_stream
    for out in OUTS:
        p = plan(fq, m, n, kp, _lib.I8, b_code, code[out])
        assert p.kernel == kern, (path, out, p.kernel)
        if packed and kern == 2:
            assert p.tile_m == 512, (path, out, p.tile_m)
        if tile_n is not None:
            assert p.tile_n == tile_n, (path, out, p.tile_n)
        assert (p.splits > 1) == split, (path, out, p.splits)
        for bias_dt in BIASES:
            if bias_dt is None:
                bias, bias_d = np.zeros(n), None
            else:
                bias = np.random.default_rng(n).standard_normal(n) * 3.0
                bias_d = torch.from_numpy(bias).to(tdt[bias_dt]).cuda()
                bias = bias_d.double().cpu().numpy()  # the bias values the device sees
            want = _round_out(acc.astype(np.float64) * s + bias[None, :], out)
            y = torch.empty((m, n), dtype=tdt[out], device="cuda")
            fq.check(fq.lib().fqg_gemm(ad.data_ptr(), _lib.I8, kp, bd.data_ptr(), b_code, ldb, m,
                                       n, kp, y.data_ptr(), code[out], n, scale.data_ptr(),
                                       bias_d.data_ptr() if bias_d is not None else None,
                                       code[bias_dt] if bias_dt else _lib.NONE, st))
            got = y.double().cpu().numpy()
            bad = np.argwhere(got != want)
            assert bad.size == 0, (f"{path} out={out} bias={bias_dt}: {len(bad)} mismatches, "
                                   f"e.g. {tuple(bad[0])}: {got[tuple(bad[0])]} vs "
                                   f"{want[tuple(bad[0])]}")


@pytest.mark.skipif(os.environ.get("FQG_GEMM_DEBUG") == "128", reason="already the child run")
def test_splitk_orphaned_chunks():
    """Split-K with no waiting at all: every split but the last writes its own
    chunks too and leaves; the last split reduces them. Same bits as the normal
    path (run in a child process: the debug bits are read once per process)."""
    env = dict(os.environ, FQG_GEMM_DEBUG="128")
    r = subprocess.run([sys.executable, "-m", "pytest", __file__, "-q", "-m", "gpu", "-x",
                        "-k", "splitk and not orphaned", "-p", "no:cacheprovider"],
                       env=env, capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stdout[-3000:] + r.stderr[-3000:]
    assert " passed" in r.stdout, r.stdout[-2000:]


@pytest.mark.parametrize("m", [1, 2, 4])
def test_layer_decode_rows_int4_weights(port, fq, m):
    """Decode-size M through the layer with biased int4 weights (tensor-core path)."""
    import torch

    from conftest import bf16_round

    k, n = 1024, 1000
    w, calib, x = fq.synthetic_layer(5, test_rows=m, in_channels=k, out_channels=n, rows=32,
                                     samples=4)
    L = port.quantize_layer(w, calib, 4)
    x = bf16_round(x)
    px = fq.FlattenPlan.from_extensions(L.t_x, L.e_x, L.block)
    pw = fq.FlattenPlan.from_extensions(L.t_w, L.e_w, L.block)
    cfg = fq.LayerQuantConfig(bits=4, smooth_scales=L.s, plan_x=px, plan_w=pw,
                              act_scale=L.act_scale, weight_q=L.wq, w_scale=L.s_w)
    layer = fq.Layer(cfg, a_format=fq.I8, b_format=fq.I4)
    y_ref, _ = port.run_layer(L, x)
    xt = torch.from_numpy(x).to(torch.bfloat16).cuda()
    y = layer.forward(xt, out_dtype=torch.float64).cpu().numpy()
    assert np.array_equal(y, y_ref)


@pytest.mark.parametrize("out", ["f16", "bf16", "f32"])
def test_layer_forward_with_bias(port, fq, out):
    """Through the layer (int4 biased weights, row-sum correction) with a bias."""
    import torch

    from conftest import bf16_round

    k, n, m = 1024, 1536, 512
    w, calib, x = fq.synthetic_layer(3, test_rows=m, in_channels=k, out_channels=n, rows=32,
                                     samples=4)
    L = port.quantize_layer(w, calib, 4)
    x = bf16_round(x)
    px = fq.FlattenPlan.from_extensions(L.t_x, L.e_x, L.block)
    pw = fq.FlattenPlan.from_extensions(L.t_w, L.e_w, L.block)
    cfg = fq.LayerQuantConfig(bits=4, smooth_scales=L.s, plan_x=px, plan_w=pw,
                              act_scale=L.act_scale, weight_q=L.wq, w_scale=L.s_w)
    layer = fq.Layer(cfg, a_format=fq.I8, b_format=fq.I4)
    y_ref, _ = port.run_layer(L, x)
    bias_t = torch.from_numpy(np.linspace(-2.0, 2.0, n)).to(torch.float32).cuda()
    bias = bias_t.double().cpu().numpy()
    tdt = {"f16": torch.float16, "bf16": torch.bfloat16, "f32": torch.float32}[out]
    xt = torch.from_numpy(x).to(torch.bfloat16).cuda()
    y = layer.forward(xt, out_dtype=tdt, bias=bias_t).double().cpu().numpy()
    assert np.array_equal(y, _round_out(y_ref + bias[None, :], out))
