"""Developer probe: K4 GEMM correctness (exact INT32 vs int64 CPU) and timing."""
import ctypes as C
import sys
import time

import numpy as np
import torch

sys.path.insert(0, __file__.rsplit("/tools/", 1)[0])
from paper_2402_17985_b200 import _lib as fl  # noqa: E402

L = fl.lib()
dev = torch.device("cuda:0")


def gemm(a, b, y_dtype, scale=None, bias=None, bias_dt=fl.NONE, kp=None):
    m, lda = a.shape
    n, ldb = b.shape
    kp = kp or lda
    tdt = {fl.I32: torch.int32, fl.F16: torch.float16, fl.F64: torch.float64,
           fl.BF16: torch.bfloat16, fl.F32: torch.float32}[y_dtype]
    y = torch.full((m, n), -7, dtype=tdt, device=dev)
    if scale is None:
        scale = torch.tensor([1.0, 1.0, 1.0], dtype=torch.float64, device=dev)
    fl.check(L.fqg_gemm(a.data_ptr(), fl.I8, lda, b.data_ptr(), fl.I8, ldb, m, n, kp, y.data_ptr(),
                        y_dtype, n, scale.data_ptr(), bias.data_ptr() if bias is not None else None,
                        bias_dt, torch.cuda.current_stream().cuda_stream))
    return y


def check_exact(m, n, k, lo=-127, hi=127):
    g = torch.Generator().manual_seed(m * 7 + n * 3 + k)
    a = torch.randint(lo, hi + 1, (m, k), generator=g, dtype=torch.int8)
    b = torch.randint(lo, hi + 1, (n, k), generator=g, dtype=torch.int8)
    ref = a.long() @ b.long().T
    y = gemm(a.to(dev), b.to(dev), fl.I32)
    torch.cuda.synchronize()
    ok = torch.equal(y.cpu().long(), ref)
    bad = (y.cpu().long() != ref).sum().item()
    print(f"exact i32 m={m} n={n} k={k}: {'OK' if ok else 'MISMATCH'} bad={bad}", flush=True)
    if not ok:
        yy = y.cpu().long()
        idx = (yy != ref).nonzero()[:5]
        for i, j in idx.tolist():
            print("   ", i, j, yy[i, j].item(), ref[i, j].item())
    return ok


def check_scaled():
    m, n, k = 300, 520, 384
    a = torch.randint(-7, 8, (m, k), dtype=torch.int8)
    b = torch.randint(-127, 128, (n, k), dtype=torch.int8)
    acc = (a.long() @ b.long().T).double()
    sx, sw = 0.01234567, 0.00078125
    s = torch.tensor([sx, sw, sx * sw], dtype=torch.float64)
    ref = acc * (sx * sw)
    y64 = gemm(a.to(dev), b.to(dev), fl.F64, s.to(dev)).cpu()
    y16 = gemm(a.to(dev), b.to(dev), fl.F16, s.to(dev)).cpu()
    bias = torch.randn(n, dtype=torch.float32)
    yb = gemm(a.to(dev), b.to(dev), fl.BF16, s.to(dev), bias.to(dev), fl.F32).cpu()
    print("f64 exact:", torch.equal(y64, ref),
          "f16 == fp16(ref):", torch.equal(y16, ref.half()),
          "bf16+bias == bf16(ref+bias):", torch.equal(yb, (ref + bias.double()).bfloat16()),
          flush=True)


def bench(m, n, k, iters=20):
    a = torch.randint(-127, 128, (m, k), dtype=torch.int8, device=dev)
    b = torch.randint(-127, 128, (n, k), dtype=torch.int8, device=dev)
    s = torch.tensor([1e-3, 1e-3, 1e-6], dtype=torch.float64, device=dev)
    for _ in range(3):
        gemm(a, b, fl.F16, s)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(iters):
        gemm(a, b, fl.F16, s)
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / iters
    tops = 2 * m * n * k / ms / 1e9
    print(f"bench m={m} n={n} k={k}: {ms*1e3:.1f} us  {tops:.0f} TOPS", flush=True)


if __name__ == "__main__":
    print(torch.cuda.get_device_name(0), flush=True)
    ok = True
    ok &= check_exact(128, 256, 128)
    ok &= check_exact(200, 300, 160)
    ok &= check_exact(1000, 1024, 7296)
    ok &= check_exact(37, 4096, 512)
    ok &= check_exact(513, 1728, 7104)
    check_scaled()
    if ok:
        bench(2048, 4096, 7296)
        bench(4096, 4096, 7296)
        bench(8192, 8192, 8192)
        bench(256, 4096, 7296)
