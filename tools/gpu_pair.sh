echo "== variant 1"; FQG_GEMM_VARIANT=1 timeout 300 python tools/probe_gemm.py 2>&1 | tail -12
echo "== variant 2"; FQG_GEMM_VARIANT=2 timeout 300 python tools/probe_gemm.py 2>&1 | tail -12
echo "== parity (variant 2)"; FQG_GEMM_VARIANT=2 timeout 600 python -m pytest tests/test_gpu_parity.py -x -q 2>&1 | tail -4
