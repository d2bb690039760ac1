timeout 900 python -m pytest tests/test_gpu_epilogue.py tests/test_gpu_full.py -x -q 2>&1 | tail -2
FQG_GEMM_DEBUG=1 timeout 120 python tools/layer_gemm_dbg.py 2>&1 | grep -E "accumulator ready|per CTA: mma|per leader" | tail -3
bash tools/gpu_ab.sh
