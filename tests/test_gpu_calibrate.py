"""§8f row 3: fq::quantize_layer's calibration and KL bit selection on the
device (fqg_calibrate) against the UNMODIFIED reference quantize_layer
(oracle/_ref): every recipe field, the KL ratios and the chosen bit width must
be identical (bit for bit), and so must the weight_q the device weight tail
then computes and the layer outputs."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu

CASES = [  # (layer index, K, N, rows, samples, mode, gamma)
    (0, 256, 192, 32, 4, 2, 1.86),    # KL picks (the generator's layers go INT4)
    (1, 512, 384, 48, 3, 2, 0.5),     # a gamma that forces INT8 through the ratios
    (2, 384, 256, 32, 4, 1, 1.86),    # O1 pins 8 bits; ratios still recorded
    (3, 1024, 512, 64, 4, 2, 1.86),
]


@pytest.mark.parametrize("idx,k,n,rows,samples,mode,gamma", CASES)
def test_calibrate_equals_reference_quantize_layer(ref, fq, idx, k, n, rows, samples, mode,
                                                   gamma):
    w, calib, x, _ = ref.synthetic_layer(idx, in_channels=k, out_channels=n, rows=rows,
                                         samples=samples)
    rl = ref.quantize_layer(w, calib, mode=mode, gamma=gamma)
    L = rl.to_layer()
    cfg, info = fq.calibrate(w, calib, mode=mode, gamma=gamma)
    assert cfg.bits == L.bits
    assert info["kl_ratio_act"] == rl.info.kl_ratio_act
    assert info["kl_ratio_w"] == rl.info.kl_ratio_w
    assert np.array_equal(cfg.smooth_scales, L.s)
    assert cfg.plan_x.threshold == L.t_x and cfg.plan_w.threshold == L.t_w
    assert np.array_equal(cfg.plan_x.extensions, L.e_x)
    assert np.array_equal(cfg.plan_w.extensions, L.e_w)
    assert cfg.act_scale == L.act_scale and info["w_scale"] == L.s_w
    layer = fq.Layer(cfg, b_format=fq.I4 if cfg.bits == 4 else fq.I8)
    assert layer.w_scale == L.s_w
    assert np.array_equal(layer.weight_q(), L.wq)
    y_ref, sat_ref = rl.run_layer(x)
    y, sat = layer.run_layer(x)
    assert np.array_equal(y, y_ref) and sat == sat_ref


def test_calibrate_options_and_errors(ref, fq):
    w, calib, _, _ = ref.synthetic_layer(4, in_channels=128, out_channels=96, rows=16, samples=2)
    for smooth, clip, bins in ((0, 1, 2048), (1, 0, 512), (0, 0, 64)):
        rl = ref.quantize_layer(w, calib, mode=2, smooth=smooth, clip=clip, bins=bins)
        cfg, info = fq.calibrate(w, calib, mode=2, smooth=smooth, clip=clip, bins=bins)
        assert cfg.bits == rl.info.bits and info["kl_ratio_act"] == rl.info.kl_ratio_act
        assert cfg.plan_x.threshold == rl.info.T_x
    with pytest.raises(fq.FqgInvalidArgument):
        fq.calibrate(w, calib, mode=2, bins=8)


@pytest.mark.parametrize("idx,k,n,rows,samples,bits_gamma", [(5, 96, 64, 32, 4, 1e6),
                                                              (6, 160, 96, 48, 2, 0.5),
                                                              (7, 256, 128, 64, 3, 1e6)])
def test_o3_gptq_weight_q_equals_reference(ref, fq, idx, k, n, rows, samples, bits_gamma):
    """O3 (gptq.cpp:73-161) on the device: Hessian, Cholesky, inverse factor and
    the blocked column updates keep the reference's per-element FP64 sequences,
    so weight_q is identical."""
    w, calib, x, _ = ref.synthetic_layer(idx, in_channels=k, out_channels=n, rows=rows,
                                         samples=samples)
    rl = ref.quantize_layer(w, calib, mode=3, gamma=bits_gamma)
    L = rl.to_layer()
    cfg, info = fq.calibrate(w, calib, mode=3, gamma=bits_gamma)
    assert cfg.bits == L.bits and info["w_scale"] == L.s_w
    bad = np.argwhere(cfg.weight_q != L.wq)
    assert bad.size == 0, f"{len(bad)} weight_q mismatches, first {tuple(bad[0])}"
    layer = fq.Layer(cfg, b_format=fq.I4 if cfg.bits == 4 else fq.I8)
    y_ref, sat_ref = rl.run_layer(x)
    y, sat = layer.run_layer(x)
    assert np.array_equal(y, y_ref) and sat == sat_ref
