"""Times K4 variants x operand formats (CUDA events, L2 flushed between reps)."""
import os
import sys

import torch

sys.path.insert(0, __file__.rsplit("/tools/", 1)[0])
from paper_2402_17985_b200 import _lib as fl  # noqa: E402

L = fl.lib()
dev = torch.device("cuda:0")
flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)


def run(m, n, k, af, bf, reps=10):
    a = torch.randint(-7, 8, (m, k // (2 if af == fl.I4 else 1)), dtype=torch.int8, device=dev)
    b = torch.randint(-7, 8, (n, k // (2 if bf == fl.I4 else 1)), dtype=torch.int8, device=dev)
    y = torch.empty((m, n), dtype=torch.float16, device=dev)
    s = torch.tensor([1e-3, 1e-3], dtype=torch.float64, device=dev)
    st = torch.cuda.current_stream().cuda_stream

    def go():
        fl.check(L.fqg_gemm(a.data_ptr(), af, a.stride(0), b.data_ptr(), bf, b.stride(0), m, n, k,
                            y.data_ptr(), fl.F16, n, s.data_ptr(), None, fl.NONE, st))
    for _ in range(3):
        go()
    ts = []
    for _ in range(reps):
        flush.fill_(1)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        go()
        e1.record()
        torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1))
    t = sorted(ts)[len(ts) // 2]
    return t * 1e3, 2 * m * n * k / (t * 1e-3) / 1e12


if __name__ == "__main__":
    shapes = [(2048, 4096, 7488), (256, 4096, 7488), (8192, 8192, 8192)]
    names = {fl.I8: "i8", fl.I4: "i4"}
    for (m, n, k) in shapes:
        for af, bf in ((fl.I8, fl.I8), (fl.I8, fl.I4), (fl.I4, fl.I4)):
            us, tops = run(m, n, k, af, bf)
            print(f"variant={os.environ.get('FQG_GEMM_VARIANT', 'auto')} m={m} n={n} k={k} "
                  f"A={names[af]} B={names[bf]}: {us:7.1f} us {tops:6.0f} TOPS", flush=True)
