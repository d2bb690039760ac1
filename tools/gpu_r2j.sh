timeout 900 python -m pytest tests/test_model_io.py tests/test_gpu_calibrate.py tests/test_gpu_contracts.py tests/test_gpu_epilogue.py -x -q 2>&1 | tail -5
