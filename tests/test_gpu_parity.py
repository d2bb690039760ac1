"""GPU parity: the sm_100a path vs the CPU oracle, through the C ABI.

Bar (BASELINE.json north_star): bit-exact for the flatten map, the quantized
integer tensors, the saturation count and the INT32 accumulators; the f64
output of the drop-in call equals the reference bit for bit; fp16/bf16 outputs
equal the correctly rounded reference value, hence within 1e-3 relative
(fp16) / one bf16 ulp.
"""
import numpy as np
import pytest

from conftest import bf16_round

pytestmark = pytest.mark.gpu

FP16_RTOL = 1e-3


def to_cfg(fq, L, weight=None):
    px = fq.FlattenPlan.from_extensions(L.t_x, L.e_x, L.block)
    pw = fq.FlattenPlan.from_extensions(L.t_w, L.e_w, L.block)
    return fq.LayerQuantConfig(bits=L.bits, smooth_scales=L.s, plan_x=px, plan_w=pw,
                               act_scale=L.act_scale,
                               weight_q=None if weight is not None else L.wq, w_scale=L.s_w,
                               weight=weight)


def make_case(port, fq, k, n, m, bits, index=0, rows=32, samples=4, **synth):
    w, calib, x = fq.synthetic_layer(index, test_rows=m, in_channels=k, out_channels=n, rows=rows,
                                     samples=samples, **synth)
    L = port.quantize_layer(w, calib, bits)
    return w, calib, bf16_round(x), L


def unpack_i4(packed: np.ndarray) -> np.ndarray:
    """FQG_I4: per group of 32 k, byte i = q[i] & 15 | q[16 + i] << 4."""
    p = packed.view(np.uint8).astype(np.int32)
    rows, nbytes = p.shape
    g = p.reshape(rows, nbytes // 16, 16)
    out = np.concatenate([g & 15, g >> 4], axis=2).reshape(rows, nbytes * 2)
    return np.where(out >= 8, out - 16, out)


def fp16_close(y16: np.ndarray, y_ref: np.ndarray):
    y16 = y16.astype(np.float64)
    # correctly rounded reference (fp16 normal range), hence within 2^-11 relative
    assert np.array_equal(y16, y_ref.astype(np.float16).astype(np.float64))
    scale = np.maximum(np.abs(y_ref), 1e-2)
    assert np.max(np.abs(y16 - y_ref) / scale) <= FP16_RTOL


CASES = [  # (K, N, M, bits)
    (256, 128, 64, 8),
    (256, 128, 64, 4),
    (512, 384, 200, 8),
    (384, 520, 131, 4),
    (1024, 1024, 257, 8),
]


@pytest.mark.parametrize("k,n,m,bits", CASES)
def test_quantized_activations_bit_exact(port, fq, k, n, m, bits):
    import torch

    w, calib, x, L = make_case(port, fq, k, n, m, bits)
    y_ref, sat_ref, qx_ref, acc_ref = port.run_layer(L, x, debug=True)
    for a_fmt in ([fq.I8, fq.I4] if bits == 4 else [fq.I8]):
        layer = fq.Layer(to_cfg(fq, L), a_format=a_fmt, b_format=fq.I8)
        xt = torch.from_numpy(x).to(torch.bfloat16).cuda()
        sat = torch.zeros(1, dtype=torch.int64, device="cuda")
        q = layer.quantize_acts(xt, saturation=sat).cpu().numpy()
        q = unpack_i4(q) if a_fmt == fq.I4 else q.astype(np.int32)
        assert np.array_equal(q, qx_ref), f"q_x mismatch ({(q != qx_ref).sum()} entries)"
        assert int(sat.item()) == sat_ref


@pytest.mark.parametrize("k,n,m,bits", CASES)
def test_accumulators_and_outputs(port, fq, k, n, m, bits):
    import torch

    w, calib, x, L = make_case(port, fq, k, n, m, bits, index=1)
    y_ref, sat_ref, qx_ref, acc_ref = port.run_layer(L, x, debug=True)
    fmts = [(fq.I8, fq.I8)] + ([(fq.I8, fq.I4), (fq.I4, fq.I4), (fq.I4, fq.I8)] if bits == 4 else [])
    xt = torch.from_numpy(x).to(torch.bfloat16).cuda()
    for a_fmt, b_fmt in fmts:
        layer = fq.Layer(to_cfg(fq, L), a_format=a_fmt, b_format=b_fmt)
        acc = layer.forward(xt, out_dtype=torch.int32).cpu().numpy()
        assert np.array_equal(acc.astype(np.int64), acc_ref), (a_fmt, b_fmt)
        y64 = layer.forward(xt, out_dtype=torch.float64).cpu().numpy()
        assert np.array_equal(y64, y_ref), (a_fmt, b_fmt)
        y16 = layer.forward(xt, out_dtype=torch.float16).cpu().numpy()
        fp16_close(y16, y_ref)


@pytest.mark.parametrize("bits", [8, 4])
def test_drop_in_run_layer_host_f64(port, fq, bits):
    w, calib, x, L = make_case(port, fq, 512, 256, 96, bits, index=2)
    y_ref, sat_ref = port.run_layer(L, x)
    y, sat = fq.Layer(to_cfg(fq, L)).run_layer(x)
    assert np.array_equal(y, y_ref) and sat == sat_ref


@pytest.mark.parametrize("bits", [8, 4])
def test_saturation_events_counted(port, fq, bits):
    w, calib, x, L = make_case(port, fq, 256, 128, 64, bits, index=3)
    x = x * 4.0  # far beyond the calibrated capacity of many channels
    y_ref, sat_ref = port.run_layer(L, x)
    assert sat_ref > 0
    y, sat = fq.Layer(to_cfg(fq, L)).run_layer(x)
    assert sat == sat_ref and np.array_equal(y, y_ref)


@pytest.mark.parametrize("bits,b_fmt", [(8, 5), (4, 5), (4, 6)])
def test_offline_weight_tail_bit_exact(port, fq, bits, b_fmt):
    """K3: scale_rows -> repeat_channels -> flatten_rows -> absmax -> RTN on device."""
    w, calib, x, L = make_case(port, fq, 512, 384, 64, bits, index=4)
    layer = fq.Layer(to_cfg(fq, L, weight=w), b_format=b_fmt)
    assert layer.w_scale == L.s_w
    assert np.array_equal(layer.weight_q(), L.wq)
    y_ref, _ = port.run_layer(L, x)
    y, _ = layer.run_layer(x)
    assert np.array_equal(y, y_ref)


def test_recipe_builder_matches_oracle(port, fq):
    w, calib, x, L = make_case(port, fq, 384, 200, 16, 8, index=5)
    cfg = fq.quantize_layer(w, calib, 8)
    assert cfg.plan_x.threshold == L.t_x and cfg.plan_w.threshold == L.t_w
    assert np.array_equal(cfg.smooth_scales, L.s)
    assert np.array_equal(cfg.plan_x.extensions, L.e_x)
    assert np.array_equal(cfg.plan_w.extensions, L.e_w)
    assert cfg.act_scale == L.act_scale
    layer = fq.Layer(cfg)
    assert np.array_equal(layer.weight_q(), L.wq) and layer.w_scale == L.s_w


def test_sharded_columns_are_exact_slices(port, fq):
    import torch

    w, calib, x, L = make_case(port, fq, 512, 640, 80, 8, index=6)
    y_ref, _ = port.run_layer(L, x)
    xt = torch.from_numpy(x).to(torch.bfloat16).cuda()
    parts = []
    bounds = [0, 160, 352, 640]  # uneven shards, global s_w
    for b0, b1 in zip(bounds[:-1], bounds[1:]):
        layer = fq.Layer(to_cfg(fq, L, weight=w), n_begin=b0, n=b1 - b0)
        assert layer.w_scale == L.s_w
        parts.append(layer.forward(xt, out_dtype=torch.float64).cpu().numpy())
    assert np.array_equal(np.concatenate(parts, axis=1), y_ref)


def test_dynamic_scale_mode(port, fq):
    """Opt-in dynamic per-tensor absmax (quantize.cpp:34-40 without override)."""
    import torch

    w, calib, x, L = make_case(port, fq, 256, 256, 48, 8, index=7)
    flat, _ = port.flatten_columns(x / L.s[None, :], L.t_x, L.e_x)
    rep = port.repeat_columns(flat, L.e_w)
    q_ref, s_dyn = port.quantize(rep, L.bits)
    acc_ref = port.int_matmul_raw(q_ref, L.wq)
    y_ref = acc_ref.astype(np.float64) * (s_dyn * L.s_w)
    layer = fq.Layer(to_cfg(fq, L), scale_mode=fq.SCALE_DYNAMIC)
    xt = torch.from_numpy(x).to(torch.bfloat16).cuda()
    acc = layer.forward(xt, out_dtype=torch.int32).cpu().numpy()
    assert np.array_equal(acc.astype(np.int64), acc_ref)
    y = layer.forward(xt, out_dtype=torch.float64).cpu().numpy()
    assert np.array_equal(y, y_ref)


def test_edge_cases(port, fq):
    import torch

    w, calib, x, L = make_case(port, fq, 256, 136, 8, 8, index=8)
    layer = fq.Layer(to_cfg(fq, L))
    # zero input -> zero output (test_pipeline.cpp:107-113)
    y, sat = layer.run_layer(np.zeros((3, 256)))
    assert not y.any() and sat == 0
    # M = 1 and ragged M
    for m in (1, 127, 129):
        xm = bf16_round(np.random.default_rng(m).standard_normal((m, 256)) * 3)
        y_ref, s_ref = port.run_layer(L, xm)
        y, s = layer.run_layer(xm)
        assert np.array_equal(y, y_ref) and s == s_ref
    # channel-count validation (test_pipeline.cpp:115-120)
    with pytest.raises(fq.FqgInvalidArgument):
        layer.run_layer(np.zeros((3, 257)))
    with pytest.raises(ValueError):
        layer.forward(torch.zeros((3, 255), device="cuda"))


def test_identity_plan_and_signed_zero(port, fq):
    """Thresholds above every maximum: flatten is the identity (test_flatten.cpp:38-44)."""
    rng = np.random.default_rng(11)
    k, n, m = 96, 64, 40
    w = rng.standard_normal((k, n))
    calib = rng.standard_normal((2, 16, k))
    L = port.quantize_layer(w, calib, 8, beta=50.0, smooth=False)
    assert int(L.e_x.sum()) == 0
    x = bf16_round(rng.standard_normal((m, k)))
    x[0, :5] = -0.0
    y_ref, s_ref = port.run_layer(L, x)
    y, s = fq.Layer(to_cfg(fq, L)).run_layer(x)
    assert np.array_equal(y, y_ref) and s == s_ref


def test_against_unmodified_reference(ref, fq):
    """The real fq::quantize_layer recipe and fq::run_layer, through the drop-in."""
    w, calib, x, _ = ref.synthetic_layer(0, in_channels=512, out_channels=256, rows=32, samples=4)
    for mode, gamma in ((1, 1.86), (2, 1e6)):
        rl = ref.quantize_layer(w, calib, mode=mode, gamma=gamma)
        L = rl.to_layer()
        y_ref, sat_ref = rl.run_layer(x)
        y, sat = fq.Layer(to_cfg(fq, L)).run_layer(x)
        assert np.array_equal(y, y_ref) and sat == sat_ref


@pytest.mark.slow
@pytest.mark.parametrize("bits,a_fmt,b_fmt", [(8, 5, 5), (4, 5, 6), (4, 6, 6)])
def test_full_size_row_subset(port, fq, bits, a_fmt, b_fmt):
    """BASELINE configs[0]/[1] (4096x4096, M=2048): full GPU run, oracle on a
    random row subset (rows are independent under the static scale)."""
    import torch

    k = n = 4096
    m = 2048
    w, calib, x = fq.synthetic_layer(0, test_rows=m, in_channels=k, out_channels=n, rows=32,
                                     samples=4)
    L = port.quantize_layer(w, calib, bits)
    x = bf16_round(x)
    layer = fq.Layer(to_cfg(fq, L, weight=w), a_format=a_fmt, b_format=b_fmt)
    assert layer.w_scale == L.s_w
    xt = torch.from_numpy(x).to(torch.bfloat16).cuda()
    acc = layer.forward(xt, out_dtype=torch.int32).cpu().numpy()
    y16 = layer.forward(xt, out_dtype=torch.float16).cpu().numpy()
    rows = np.sort(np.random.default_rng(bits).choice(m, 24, replace=False))
    y_ref, _, _, acc_ref = port.run_layer(L, x[rows], debug=True)
    assert np.array_equal(acc[rows].astype(np.int64), acc_ref)
    fp16_close(y16[rows], y_ref)


@pytest.mark.parametrize("m,n,kp", [(512, 10240, 1024), (2048, 4096, 512), (300, 8960, 2048),
                                    (256, 4096, 7296), (200, 1024, 4096)])
def test_gemm_stream_k_shapes(fq, m, n, kp):
    """Tile counts that leave CTA pairs idle: split-K (small M, INT32 partials
    of 2..8 clusters per tile through a workspace) and the optional stream-K
    must give the exact integer product."""
    import torch

    from paper_2402_17985_b200 import _lib

    g = torch.Generator().manual_seed(m + n)
    a = torch.randint(-127, 128, (m, kp), dtype=torch.int8, generator=g)
    b = torch.randint(-127, 128, (n, kp), dtype=torch.int8, generator=g)
    ref = a.numpy().astype(np.int64) @ b.numpy().astype(np.int64).T
    ad, bd = a.cuda(), b.cuda()
    y = torch.empty((m, n), dtype=torch.int32, device="cuda")
    fq.check(fq.lib().fqg_gemm(ad.data_ptr(), _lib.I8, kp, bd.data_ptr(), _lib.I8, kp, m, n, kp,
                               y.data_ptr(), _lib.I32, n, None, None, _lib.NONE,
                               torch.cuda.current_stream().cuda_stream))
    assert np.array_equal(y.cpu().numpy().astype(np.int64), ref)


def _rn_bf16(v):
    """Round-to-nearest-even of float64 values to bfloat16 (normal range), as float64."""
    mant, ex = np.frexp(v)
    return np.ldexp(np.round(mant * 256.0), ex - 8)


@pytest.mark.parametrize("sx,sw", [(2.0 ** -10, 1.0), (2.0 ** -14, 0.5), (3.7e-5, 0.0123),
                                   (1.0 / 3.0, 0.9), (2.0 ** -30, 1.0), (2.0 ** -3, 1.0)])
@pytest.mark.parametrize("out", ["f16", "bf16"])
@pytest.mark.parametrize("b_fmt", ["i8", "i4"])
def test_half_outputs_are_rn16_of_reference(fq, sx, sw, out, b_fmt):
    """2-byte outputs equal RN16(double(acc) * (s_x * s_w)) exactly (quantize.cpp:193-196
    rounded once). The epilogue's certified fp32 fast path must defer every element
    near a rounding midpoint: power-of-two scales make ~half of them exact ties;
    2^-30 puts outputs in the fp16 subnormal range; 0.3 straddles the fp16 maximum."""
    import torch

    from paper_2402_17985_b200 import _lib

    m, n, kp = 512, 1024, 1536
    g = torch.Generator().manual_seed(int(sx * 1e6) + n)
    a = torch.randint(-127, 128, (m, kp), dtype=torch.int8, generator=g)
    if b_fmt == "i8":  # |acc| up to 2^24.6: the split int -> float path of the epilogue
        b = torch.randint(-127, 128, (n, kp), dtype=torch.int8, generator=g)
        bdev, bcode, ldb = b.cuda(), _lib.I8, kp
    else:  # packed int4 weights, |acc| < 2^22: the one-FADD int -> float path
        b = torch.randint(-7, 8, (n, kp), dtype=torch.int8, generator=g)
        nib = (b.numpy().astype(np.int32) & 15).reshape(n, kp // 32, 2, 16)
        packed = (nib[:, :, 0, :] | (nib[:, :, 1, :] << 4)).astype(np.uint8).reshape(n, kp // 2)
        bdev, bcode, ldb = torch.from_numpy(packed.view(np.int8)).cuda(), _lib.I4, kp // 2
    acc = a.numpy().astype(np.int64) @ b.numpy().astype(np.int64).T
    v = acc.astype(np.float64) * (sx * sw)
    scale = torch.tensor([sx, sw], dtype=torch.float64, device="cuda")
    tdt = torch.float16 if out == "f16" else torch.bfloat16
    y = torch.empty((m, n), dtype=tdt, device="cuda")
    fq.check(fq.lib().fqg_gemm(a.cuda().data_ptr(), _lib.I8, kp, bdev.data_ptr(), bcode, ldb,
                               m, n, kp, y.data_ptr(), _lib.F16 if out == "f16" else _lib.BF16, n,
                               scale.data_ptr(), None, _lib.NONE,
                               torch.cuda.current_stream().cuda_stream))
    got = y.double().cpu().numpy()
    want = v.astype(np.float16).astype(np.float64) if out == "f16" else _rn_bf16(v)
    bad = np.argwhere(got != want)
    assert bad.size == 0, f"{len(bad)} mismatches, e.g. acc {acc[tuple(bad[0])]}: " \
                          f"{got[tuple(bad[0])]} vs {want[tuple(bad[0])]}"
