timeout 900 python -m pytest tests -x -q -m gpu 2>&1 | tail -5
FQG_GEMM_VARIANT=1 timeout 600 python -m pytest tests/test_gpu_parity.py -x -q 2>&1 | tail -2
timeout 120 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -2
