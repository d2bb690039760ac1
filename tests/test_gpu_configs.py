"""BASELINE.json configs as GPU parity cases (the bench measures configs[1]).

configs[2] OPT-6.7B decoder-layer linears (QKV/O/FC1/FC2) with mixed 4/8-bit
recipes, configs[3] the LLaMA-13B MLP up-projection N-sharded over 2/4/8 ranks
(shards must be exact column slices of the unsharded layer), configs[4] the
8192x8192 INT8 sweep at several M (split-K for small M, 256x512 tiles for
large). The GPU runs the full batch; the CPU oracle checks a random row subset
(rows are independent under the static scale) bit for bit on the INT32
accumulators and the fp16 outputs.
"""
import numpy as np
import pytest

from conftest import bf16_round

pytestmark = [pytest.mark.gpu, pytest.mark.slow]


def layer_case(port, fq, k, n, m, bits, index, a_fmt=None, b_fmt=None):
    import torch

    w, calib, x = fq.synthetic_layer(index, test_rows=m, in_channels=k, out_channels=n, rows=32,
                                     samples=4)
    L = port.quantize_layer(w, calib, bits)
    x = bf16_round(x)
    px = fq.FlattenPlan.from_extensions(L.t_x, L.e_x, L.block)
    pw = fq.FlattenPlan.from_extensions(L.t_w, L.e_w, L.block)
    cfg = fq.LayerQuantConfig(bits=bits, smooth_scales=L.s, plan_x=px, plan_w=pw,
                              act_scale=L.act_scale, weight_q=None, w_scale=L.s_w, weight=w)
    a_fmt = a_fmt if a_fmt is not None else fq.I8
    b_fmt = b_fmt if b_fmt is not None else (fq.I4 if bits == 4 else fq.I8)
    return L, cfg, x, torch.from_numpy(x).to(torch.bfloat16).cuda(), a_fmt, b_fmt


def check_rows(port, L, x, acc, y16, rows):
    y_ref, _, _, acc_ref = port.run_layer(L, x[rows], debug=True)
    assert np.array_equal(acc[rows].astype(np.int64), acc_ref)
    assert np.array_equal(y16[rows].astype(np.float64), y_ref.astype(np.float16).astype(np.float64))


@pytest.mark.parametrize("name,k,n,bits", [("qkv", 4096, 12288, 4), ("o", 4096, 4096, 8),
                                           ("fc1", 4096, 16384, 4), ("fc2", 16384, 4096, 8)])
def test_opt67b_linears(port, fq, name, k, n, bits):
    import torch

    m = 512
    L, cfg, x, xt, a_fmt, b_fmt = layer_case(port, fq, k, n, m, bits, index=len(name))
    layer = fq.Layer(cfg, a_format=a_fmt, b_format=b_fmt)
    assert np.array_equal(layer.weight_q(), L.wq)
    acc = layer.forward(xt, out_dtype=torch.int32).cpu().numpy()
    y16 = layer.forward(xt, out_dtype=torch.float16).cpu().numpy()
    rows = np.sort(np.random.default_rng(k + n).choice(m, 12, replace=False))
    check_rows(port, L, x, acc, y16, rows)


@pytest.mark.parametrize("world", [2, 4, 8])
def test_llama13b_up_shards_are_exact(port, fq, world):
    import torch

    from paper_2402_17985_b200.shard import shard_bounds

    k, n, m = 5120, 13824, 256
    L, cfg, x, xt, a_fmt, b_fmt = layer_case(port, fq, k, n, m, 4, index=13)
    full = fq.Layer(cfg, a_format=a_fmt, b_format=b_fmt)
    y_full = full.forward(xt, out_dtype=torch.int32).cpu().numpy()
    parts = []
    for r in range(world):
        b0, b1 = shard_bounds(n, world, r)
        shard = fq.Layer(cfg, a_format=a_fmt, b_format=b_fmt, n_begin=b0, n=b1 - b0)
        assert shard.w_scale == full.w_scale  # global s_w
        parts.append(shard.forward(xt, out_dtype=torch.int32).cpu().numpy())
    assert np.array_equal(np.concatenate(parts, axis=1), y_full)
    y16 = full.forward(xt, out_dtype=torch.float16).cpu().numpy()
    rows = np.sort(np.random.default_rng(world).choice(m, 8, replace=False))
    check_rows(port, L, x, y_full, y16, rows)


@pytest.mark.parametrize("m", [1, 7, 64, 300, 2048])
def test_sweep_8192_int8(port, fq, m):
    import torch

    k = n = 8192
    L, cfg, x, xt, a_fmt, b_fmt = layer_case(port, fq, k, n, m, 8, index=21)
    layer = fq.Layer(cfg, a_format=a_fmt, b_format=b_fmt)
    acc = layer.forward(xt, out_dtype=torch.int32).cpu().numpy()
    y16 = layer.forward(xt, out_dtype=torch.float16).cpu().numpy()
    rows = np.sort(np.random.default_rng(m).choice(m, min(m, 6), replace=False))
    check_rows(port, L, x, acc, y16, rows)


def test_llama13b_up_full_batch_int4(port, fq):
    """configs[3] at M = 2048 on one GPU: 216 tiles of 256 x 512 on 74 CTA pairs
    (several tiles per pair with the single-accumulator epilogue and int4 unpack)."""
    import torch

    k, n, m = 5120, 13824, 2048
    L, cfg, x, xt, a_fmt, b_fmt = layer_case(port, fq, k, n, m, 4, index=13)
    layer = fq.Layer(cfg, a_format=a_fmt, b_format=b_fmt)
    acc = layer.forward(xt, out_dtype=torch.int32).cpu().numpy()
    y16 = layer.forward(xt, out_dtype=torch.float16).cpu().numpy()
    rows = np.sort(np.random.default_rng(5).choice(m, 8, replace=False))
    check_rows(port, L, x, acc, y16, rows)
