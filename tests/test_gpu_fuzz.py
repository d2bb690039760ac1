"""Randomised K4 parity: fqg_gemm on random shapes / formats / outputs / bias against the exact
product (every kernel path the planner can pick: CUDA-core decode rows, 1-CTA, CTA-pair tiles,
split-K with its fix-up). FQG_FUZZ_CASES raises the case count (default 24)."""
import ctypes as C
import os

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def _round_out(v, out):
    if out == "f16":
        return v.astype(np.float16).astype(np.float64)
    if out == "bf16":
        mant, ex = np.frexp(v)
        return np.ldexp(np.round(mant * 256.0), ex - 8)
    if out == "f32":
        return v.astype(np.float32).astype(np.float64)
    return v


CASES = int(os.environ.get("FQG_FUZZ_CASES", "24"))


@pytest.mark.parametrize("case", range(CASES))
def test_gemm_fuzz(fq, case):
    import torch

    from paper_2402_17985_b200 import _lib

    rng = np.random.default_rng(1000 + case)
    m = int(rng.choice([1, 2, 3, 5, 17, 64, 100, 256, 300, 511, 777, 1024, 2048]))
    n = int(rng.integers(1, 160)) * 32
    kp = int(rng.integers(1, 96)) * 32
    packed = bool(rng.integers(0, 2))
    out = str(rng.choice(["f16", "bf16", "f32", "f64", "i32"]))
    bias_dt = None if out == "i32" or rng.integers(0, 2) else str(rng.choice(["f64", "f32", "f16", "bf16"]))
    g = torch.Generator().manual_seed(case)
    a = torch.randint(-127, 128, (m, kp), dtype=torch.int8, generator=g)
    b = torch.randint(-7 if packed else -127, 8 if packed else 128, (n, kp), dtype=torch.int8,
                      generator=g)
    # exact in f64 BLAS: every partial sum is an integer below 2^53
    acc = (a.numpy().astype(np.float64) @ b.numpy().astype(np.float64).T).astype(np.int64)
    if packed:  # FQG_I4: per group of 32 k, byte i = q[i] & 15 | q[16 + i] << 4
        nib = (b.numpy().astype(np.int32) & 15).reshape(n, kp // 32, 2, 16)
        b = torch.from_numpy((nib[:, :, 0, :] | (nib[:, :, 1, :] << 4)).astype(np.uint8)
                             .reshape(n, kp // 2).view(np.int8))
    b_code, ldb = (_lib.I4, kp // 2) if packed else (_lib.I8, kp)
    sx, sw = float(rng.uniform(1e-5, 1e-2)), float(rng.uniform(1e-4, 5e-2))
    s = sx * sw
    scale = torch.tensor([sx, sw], dtype=torch.float64, device="cuda")
    tdt = {"f16": torch.float16, "bf16": torch.bfloat16, "f32": torch.float32,
           "f64": torch.float64, "i32": torch.int32}
    code = {"f16": _lib.F16, "bf16": _lib.BF16, "f32": _lib.F32, "f64": _lib.F64, "i32": _lib.I32}
    if bias_dt is None:
        bias, bias_d = np.zeros(n), None
    else:
        bias_d = torch.from_numpy(rng.standard_normal(n) * 2.0).to(tdt[bias_dt]).cuda()
        bias = bias_d.double().cpu().numpy()
    y = torch.empty((m, n), dtype=tdt[out], device="cuda")
    info = _lib.GemmPlan()
    fq.check(fq.lib().fqg_gemm_plan(m, n, kp, _lib.I8, b_code, code[out], C.byref(info)))
    ad, bd = a.cuda(), b.cuda()  # (kept alive: a temporary's memory could be reused at once)
    fq.check(fq.lib().fqg_gemm(ad.data_ptr(), _lib.I8, kp, bd.data_ptr(), b_code, ldb, m,
                               n, kp, y.data_ptr(), code[out], n, scale.data_ptr(),
                               bias_d.data_ptr() if bias_d is not None else None,
                               code[bias_dt] if bias_dt else _lib.NONE,
                               torch.cuda.current_stream().cuda_stream))
    got = y.cpu().numpy().astype(np.int64) if out == "i32" else y.double().cpu().numpy()
    want = acc if out == "i32" else _round_out(acc.astype(np.float64) * s + bias[None, :], out)
    bad = np.argwhere(got != want)
    assert bad.size == 0, (f"case {case}: m={m} n={n} kp={kp} packed={packed} out={out} "
                           f"bias={bias_dt} plan=(kernel {info.kernel}, {info.tile_m}x{info.tile_n}, "
                           f"splits {info.splits}): {len(bad)} mismatches, first {tuple(bad[0])}")
