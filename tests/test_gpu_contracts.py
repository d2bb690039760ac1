"""GPU contract tests from the round-1 code review:

* plan block widths whose padded widths are not multiples of 32 are refused
  with FQG_ERR_UNSUPPORTED before anything is packed or uploaded;
* the general K1 (f32/f64 inputs, used by the drop-in run_host) clamps to
  +-qmax when act_scale * qmax < T_x (quantize.cpp:44-45), like the reference;
* the dynamic-scale mode through run_host is ONE per-tensor absmax over all M
  rows (quantize.cpp:34-40), not one per row chunk.
"""
import dataclasses

import numpy as np
import pytest

from conftest import bf16_round

pytestmark = pytest.mark.gpu


def _cfg(fq, L):
    px = fq.FlattenPlan.from_extensions(L.t_x, L.e_x, L.block)
    pw = fq.FlattenPlan.from_extensions(L.t_w, L.e_w, L.block)
    return fq.LayerQuantConfig(bits=L.bits, smooth_scales=L.s, plan_x=px, plan_w=pw,
                               act_scale=L.act_scale, weight_q=L.wq, w_scale=L.s_w)


def test_block16_refused_cleanly(fq):
    """block 16 with 20 extension slots: K' = 144, not a multiple of 32."""
    from paper_2402_17985_b200 import _lib

    k, n = 112, 64
    e_x = np.zeros(k, np.int64)
    e_x[0] = 20
    px = fq.FlattenPlan.from_extensions(1.0, e_x, 16)
    pw = fq.FlattenPlan.from_extensions(1.0, np.zeros(px.padded_width, np.int64), 16)
    assert px.padded_width % 32 == 16 and pw.padded_width % 32 == 16
    cfg = fq.LayerQuantConfig(bits=4, smooth_scales=np.ones(k), plan_x=px, plan_w=pw,
                              act_scale=1.0 / 7, weight_q=np.zeros((pw.padded_width, n), np.int32),
                              w_scale=1.0)
    for a_fmt, b_fmt in ((fq.I4, fq.I4), (fq.I8, fq.I8)):
        with pytest.raises(_lib.FqgError) as ei:
            fq.Layer(cfg, a_format=a_fmt, b_format=b_fmt)
        assert ei.value.code == _lib.ERR_UNSUPPORTED


@pytest.mark.parametrize("bits", [8, 4])
def test_general_k1_clamps_when_act_scale_below_threshold(port, fq, bits):
    """act_scale = T_x / (2 qmax): tier-1 values reach 2 qmax and must clamp."""
    w, calib, x = fq.synthetic_layer(1, test_rows=96, in_channels=256, out_channels=128, rows=32,
                                     samples=4)
    L = port.quantize_layer(w, calib, bits)
    qmax = (1 << (bits - 1)) - 1
    L2 = dataclasses.replace(L, act_scale=L.t_x / (2 * qmax))
    y_ref, sat_ref = port.run_layer(L2, x)  # f64 input: the general K1 on the device
    layer = fq.Layer(_cfg(fq, L2))
    y, sat = layer.run_layer(x)
    assert sat == sat_ref
    assert np.array_equal(y, y_ref)


def test_dynamic_scale_run_host_is_one_tensor_absmax(port, fq):
    """M = 300 > the 128-row chunks of run_host: one s_x for the whole input."""
    w, calib, x = fq.synthetic_layer(7, test_rows=300, in_channels=256, out_channels=192, rows=32,
                                     samples=4)
    L = port.quantize_layer(w, calib, 8)
    x = bf16_round(x)
    flat, _ = port.flatten_columns(x / L.s[None, :], L.t_x, L.e_x)
    rep = port.repeat_columns(flat, L.e_w)
    q_ref, s_dyn = port.quantize(rep, L.bits)
    acc_ref = port.int_matmul_raw(q_ref, L.wq)
    y_ref = acc_ref.astype(np.float64) * (s_dyn * L.s_w)
    layer = fq.Layer(_cfg(fq, L), scale_mode=fq.SCALE_DYNAMIC)
    y, _ = layer.run_layer(x)
    assert np.array_equal(y, y_ref)


def test_forward_sharded_c_abi_emulated_two_ranks(port, fq):
    """fqg_layer_forward_sharded: each rank's shard lands in its slot of the
    shard-major buffer and the caller's ncclAllGather-shaped collective is called
    with (this slot, the buffer, m * width, ncclFloat16). Two ranks emulated on
    one GPU share the buffer, so the collective is a recorded no-op."""
    import ctypes as C

    import torch

    from paper_2402_17985_b200 import _lib

    k, n, m, world = 1024, 1000, 384, 2
    w, calib, x = fq.synthetic_layer(4, test_rows=m, in_channels=k, out_channels=n, rows=32,
                                     samples=4)
    cfg = fq.quantize_layer(w, calib, 4)
    xt = torch.from_numpy(x).to(torch.bfloat16).cuda()
    full = fq.Layer(cfg, b_format=fq.I4).forward(xt, out_dtype=torch.float16)
    width = C.c_int64()
    fq.check(fq.lib().fqg_shard_bounds(n, world, 0, None, None, C.byref(width)))
    buf = torch.empty((world, m, width.value), dtype=torch.float16, device="cuda")
    calls = []

    @_lib.ALLGATHER_FN
    def fake_allgather(send, recv, count, dtype, comm, stream):
        calls.append((send, recv, count, dtype, comm))
        return 0

    st = torch.cuda.current_stream().cuda_stream
    for rank in range(world):
        b0, b1 = C.c_int64(), C.c_int64()
        fq.check(fq.lib().fqg_shard_bounds(n, world, rank, C.byref(b0), C.byref(b1), None))
        layer = fq.Layer(cfg, b_format=fq.I4, n_begin=b0.value, n=b1.value - b0.value)
        fq.check(fq.lib().fqg_layer_forward_sharded(
            layer._h, xt.data_ptr(), fq.BF16, m, buf.data_ptr(), fq.F16, world, rank, None,
            fq.NONE, None, fake_allgather, C.c_void_p(1234), st))
        torch.cuda.synchronize()
        slot = buf.data_ptr() + rank * m * width.value * 2
        assert calls[-1] == (slot, buf.data_ptr(), m * width.value, 6, 1234)
    y = buf.permute(1, 0, 2).reshape(m, world * width.value)[:, :n]
    assert torch.equal(y, full)
    # a layer that is not the rank's shard is refused
    wrong = fq.Layer(cfg, b_format=fq.I4, n_begin=0, n=256)
    with pytest.raises(fq.FqgError):
        fq.check(fq.lib().fqg_layer_forward_sharded(
            wrong._h, xt.data_ptr(), fq.BF16, m, buf.data_ptr(), fq.F16, world, 0, None, fq.NONE,
            None, None, None, st))
