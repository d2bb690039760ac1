"""GPU parity of the 16-bit K1 fast path (flatten16.cu) against the CPU oracle.

The fast path is selected for bf16/f16 activations under the static scale. Its
per-channel certificate (k_tier1_tables) claims bit-exactness for EVERY input;
these tests check that claim exhaustively over all 16-bit magnitudes (both
signs) on small layers, on the synthetic workload, on the queue-overflow
rescan path (every element with full pieces) and on ragged shapes.
"""
import numpy as np
import pytest

from conftest import bf16_round

pytestmark = pytest.mark.gpu


def to_cfg(fq, L):
    px = fq.FlattenPlan.from_extensions(L.t_x, L.e_x, L.block)
    pw = fq.FlattenPlan.from_extensions(L.t_w, L.e_w, L.block)
    return fq.LayerQuantConfig(bits=L.bits, smooth_scales=L.s, plan_x=px, plan_w=pw,
                               act_scale=L.act_scale, weight_q=L.wq, w_scale=L.s_w)


def unpack_i4(packed):
    p = packed.view(np.uint8).astype(np.int32)
    rows, nbytes = p.shape
    g = p.reshape(rows, nbytes // 16, 16)
    out = np.concatenate([g & 15, g >> 4], axis=2).reshape(rows, nbytes * 2)
    return np.where(out >= 8, out - 16, out)


def f16_round(x):
    return x.astype(np.float16).astype(np.float64)


def all_magnitudes(dtype: str, limit: float = 1e15) -> np.ndarray:
    """Every finite non-negative 16-bit value below `limit` (as f64)."""
    import torch

    u = np.arange(0x7C00 if dtype == "f16" else 0x7F80, dtype=np.int32).astype(np.int16)
    t = torch.from_numpy(u).view(torch.float16 if dtype == "f16" else torch.bfloat16)
    v = t.double().numpy()
    return v[v < limit]


def run_both(port, fq, L, x, dtype, a_fmt):
    import torch

    tdt = torch.bfloat16 if dtype == "bf16" else torch.float16
    layer = fq.Layer(to_cfg(fq, L), a_format=a_fmt)
    xt = torch.from_numpy(x).to(tdt).cuda()
    assert np.array_equal(xt.double().cpu().numpy(), x), "input not exactly representable"
    sat = torch.zeros(1, dtype=torch.int64, device="cuda")
    q = layer.quantize_acts(xt, saturation=sat).cpu().numpy()
    q = unpack_i4(q) if a_fmt == fq.I4 else q.astype(np.int32)
    _, sat_ref, q_ref, _ = port.run_layer(L, x, debug=True)
    return q, int(sat.item()), q_ref, sat_ref


@pytest.mark.parametrize("dtype", ["bf16", "f16"])
@pytest.mark.parametrize("bits", [8, 4])
def test_exhaustive_magnitudes(port, fq, dtype, bits):
    """Each channel sees every 16-bit magnitude below 1e15, with both signs."""
    k, n = 64, 32
    w, calib, _ = fq.synthetic_layer(3, test_rows=8, in_channels=k, out_channels=n, rows=32,
                                     samples=4)
    L = port.quantize_layer(w, calib, bits)
    mags = all_magnitudes(dtype)
    m = 2 * len(mags)
    rows = np.arange(m)
    idx = ((rows[:, None] // 2) + 37 * np.arange(k)[None, :]) % len(mags)
    x = mags[idx] * np.where(rows % 2 == 0, 1.0, -1.0)[:, None]
    for a_fmt in ([fq.I8, fq.I4] if bits == 4 else [fq.I8]):
        q, sat, q_ref, sat_ref = run_both(port, fq, L, x, dtype, a_fmt)
        bad = np.argwhere(q != q_ref)
        assert bad.size == 0, f"{len(bad)} mismatches, first at {bad[:4].tolist()}"
        assert sat == sat_ref


@pytest.mark.parametrize("dtype", ["bf16", "f16"])
@pytest.mark.parametrize("k,n,m,bits,index", [(1024, 256, 513, 8, 1), (2048, 256, 301, 4, 2),
                                              (4096, 128, 64, 4, 0)])
def test_synthetic_layers(port, fq, dtype, k, n, m, bits, index):
    w, calib, x = fq.synthetic_layer(index, test_rows=m, in_channels=k, out_channels=n, rows=32,
                                     samples=4)
    L = port.quantize_layer(w, calib, bits)
    x = bf16_round(x) if dtype == "bf16" else f16_round(np.clip(x, -6e4, 6e4))
    for a_fmt in ([fq.I8, fq.I4] if bits == 4 else [fq.I8]):
        q, sat, q_ref, sat_ref = run_both(port, fq, L, x, dtype, a_fmt)
        assert np.array_equal(q, q_ref)
        assert sat == sat_ref


@pytest.mark.parametrize("bits", [8, 4])
def test_queue_overflow_rescan(port, fq, bits):
    """Every element carries full pieces: the tier-2 queue overflows and the
    block is rescanned; saturation must still be counted once per element."""
    k, n, m = 512, 64, 37
    w, calib, _ = fq.synthetic_layer(5, test_rows=8, in_channels=k, out_channels=n, rows=32,
                                     samples=4)
    L = port.quantize_layer(w, calib, bits)
    rng = np.random.default_rng(bits)
    big = L.t_x * np.abs(L.s) * rng.uniform(1.0, 90.0, (m, k))
    x = bf16_round(big * rng.choice([-1.0, 1.0], (m, k)))
    for a_fmt in ([fq.I8, fq.I4] if bits == 4 else [fq.I8]):
        q, sat, q_ref, sat_ref = run_both(port, fq, L, x, "bf16", a_fmt)
        assert np.array_equal(q, q_ref)
        assert sat == sat_ref and sat > 0


def test_forward_matches_oracle_bf16_odd_rows(port, fq):
    """End to end (K1 fast path + K4) on an odd row count: the last block is partial."""
    import torch

    k, n, m = 768, 200, 77
    w, calib, x = fq.synthetic_layer(9, test_rows=m, in_channels=k, out_channels=n, rows=32,
                                     samples=4)
    L = port.quantize_layer(w, calib, 8)
    x = bf16_round(x)
    y_ref, _, _, acc_ref = port.run_layer(L, x, debug=True)
    layer = fq.Layer(to_cfg(fq, L))
    xt = torch.from_numpy(x).to(torch.bfloat16).cuda()
    acc = layer.forward(xt, out_dtype=torch.int32).cpu().numpy()
    assert np.array_equal(acc.astype(np.int64), acc_ref)
    y = layer.forward(xt, out_dtype=torch.float64).cpu().numpy()
    assert np.array_equal(y, y_ref)


@pytest.mark.parametrize("dtype,a_fmt_name", [("bf16", "I8"), ("bf16", "I4"), ("f32", "I8")])
def test_rowsum_and_split_entry_points(port, fq, dtype, a_fmt_name):
    """quantize_acts_ex row sums == sum of the operand row; gemm_ex with them
    (biased int4 weights) == the oracle's INT32 accumulators."""
    import torch

    a_fmt = getattr(fq, a_fmt_name)
    k, n, m = 1024, 192, 70
    w, calib, x = fq.synthetic_layer(4, test_rows=m, in_channels=k, out_channels=n, rows=32,
                                     samples=4)
    L = port.quantize_layer(w, calib, 4)
    x = bf16_round(x)
    _, _, q_ref, acc_ref = port.run_layer(L, x, debug=True)
    layer = fq.Layer(to_cfg(fq, L), a_format=a_fmt, b_format=fq.I4)
    xt = torch.from_numpy(x).to(torch.bfloat16 if dtype == "bf16" else torch.float32).cuda()
    cols = layer.kp // 2 if a_fmt == fq.I4 else layer.kp
    q = torch.empty((m, cols), dtype=torch.int8, device="cuda")
    rs = torch.empty(m, dtype=torch.int32, device="cuda")
    st = torch.cuda.current_stream().cuda_stream
    fq.check(fq.lib().fqg_layer_quantize_acts_ex(layer._h, xt.data_ptr(),
                                                 fq._lib.BF16 if dtype == "bf16" else fq._lib.F32,
                                                 m, q.data_ptr(), rs.data_ptr(), None, st))
    torch.cuda.synchronize()
    assert np.array_equal(rs.cpu().numpy().astype(np.int64), q_ref.sum(axis=1))
    acc = torch.empty((m, n), dtype=torch.int32, device="cuda")
    fq.check(fq.lib().fqg_layer_gemm_ex(layer._h, q.data_ptr(), rs.data_ptr(), m, acc.data_ptr(),
                                        fq._lib.I32, n, None, fq.NONE, st))
    assert np.array_equal(acc.cpu().numpy().astype(np.int64), acc_ref)
    acc2 = layer.gemm(q, out_dtype=torch.int32)  # row sums recomputed internally
    assert np.array_equal(acc2.cpu().numpy().astype(np.int64), acc_ref)
