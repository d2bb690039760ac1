"""Run the bench's K4 (headline layer, biased int4 weights) once with FQG_GEMM_DEBUG set.

  python tools/layer_gemm_dbg.py [b_format code] ; DBG_M / DBG_K / DBG_N / DBG_BITS override the shape."""
import os
import sys
import torch
sys.path.insert(0, __file__.rsplit("/tools/", 1)[0])
import paper_2402_17985_b200 as fq
k, n, m = (int(os.environ.get(v, d)) for v, d in (("DBG_K", 4096), ("DBG_N", 4096), ("DBG_M", 2048)))
bits = int(os.environ.get("DBG_BITS", 4))
bfmt = fq.I4 if len(sys.argv) < 2 else int(sys.argv[1])
w, calib, x = fq.synthetic_layer(0, test_rows=m, in_channels=k, out_channels=n, rows=32, samples=4)
cfg = fq.quantize_layer(w, calib, bits)
layer = fq.Layer(cfg, a_format=fq.I8, b_format=bfmt)
xt = torch.from_numpy(x).to(torch.bfloat16).cuda()
q = torch.empty((m, layer.kp), dtype=torch.int8, device="cuda")
rs = torch.empty(m, dtype=torch.int32, device="cuda")
y = torch.empty((m, n), dtype=torch.float16, device="cuda")
st = torch.cuda.current_stream().cuda_stream
fq.check(fq.lib().fqg_layer_quantize_acts_ex(layer._h, xt.data_ptr(), fq.BF16, m, q.data_ptr(), rs.data_ptr(), None, st))
flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
for i in range(3):
    flush.fill_(i)
    fq.check(fq.lib().fqg_layer_gemm_ex(layer._h, q.data_ptr(), rs.data_ptr(), m, y.data_ptr(), fq.F16, n, None, fq.NONE, st))
    torch.cuda.synchronize()
