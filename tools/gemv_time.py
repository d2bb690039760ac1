"""Time fqg_gemm at decode-size M (the CUDA-core path) against the weight bytes."""
import ctypes
import sys

import torch

sys.path.insert(0, __file__.rsplit("/tools/", 1)[0])
import paper_2402_17985_b200 as fq  # noqa: E402
from paper_2402_17985_b200 import _lib  # noqa: E402

n, kp = 8192, 14848
fl = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
st = torch.cuda.current_stream().cuda_stream
sc = torch.tensor([1e-3, 1e-3], dtype=torch.float64, device="cuda")
for bfmt, name in ((_lib.I8, "int8"), (_lib.I4, "int4")):
    ldb = kp if bfmt == _lib.I8 else kp // 2
    b = torch.randint(-127, 128, (n, ldb), dtype=torch.int8, device="cuda")
    for m in (1, 2, 4):
        a = torch.randint(-127, 128, (m, kp), dtype=torch.int8, device="cuda")
        y = torch.empty((m, n), dtype=torch.float16, device="cuda")
        info = _lib.GemmPlan()
        fq.check(fq.lib().fqg_gemm_plan(m, n, kp, _lib.I8, bfmt, _lib.F16, ctypes.byref(info)))
        ts = []
        for i in range(12):
            fl.fill_(i)
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            fq.check(fq.lib().fqg_gemm(a.data_ptr(), _lib.I8, kp, b.data_ptr(), bfmt, ldb, m, n, kp,
                                       y.data_ptr(), _lib.F16, n, sc.data_ptr(), None, _lib.NONE, st))
            e1.record()
            torch.cuda.synchronize()
            ts.append(e0.elapsed_time(e1))
        t = sorted(ts[2:])[len(ts[2:]) // 2]
        print(f"{name} M={m} kernel={info.kernel} ctas={info.ctas}: {t * 1e3:.1f} us, "
              f"weights {n * ldb / t / 1e6:.0f} GB/s")
