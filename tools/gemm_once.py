"""Run one K4 GEMM config a few times (for ncu): M N K variant a_fmt b_fmt."""
import sys
import torch
sys.path.insert(0, __file__.rsplit("/tools/", 1)[0])
from paper_2402_17985_b200 import _lib as fl
m, n, k = (int(v) for v in sys.argv[1:4])
af = int(sys.argv[4]) if len(sys.argv) > 4 else fl.I8
bf = int(sys.argv[5]) if len(sys.argv) > 5 else fl.I8
dev = torch.device("cuda:0")
a = torch.randint(-127, 128, (m, k // (2 if af == fl.I4 else 1)), dtype=torch.int8, device=dev)
b = torch.randint(-127, 128, (n, k // (2 if bf == fl.I4 else 1)), dtype=torch.int8, device=dev)
y = torch.empty((m, n), dtype=torch.float16, device=dev)
s = torch.tensor([1e-3, 1e-3], dtype=torch.float64, device=dev)
L = fl.lib()
for _ in range(5):
    fl.check(L.fqg_gemm(a.data_ptr(), af, a.stride(0), b.data_ptr(), bf, b.stride(0), m, n, k,
                        y.data_ptr(), fl.F16, n, s.data_ptr(), None, fl.NONE,
                        torch.cuda.current_stream().cuda_stream))
torch.cuda.synchronize()
