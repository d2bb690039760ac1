timeout 900 python -m pytest tests/test_gpu_k1_fast.py tests/test_gpu_parity.py tests/test_gpu_contracts.py tests/test_gpu_epilogue.py -x -q 2>&1 | tail -3
timeout 900 python -m pytest tests/test_gpu_full.py -x -q 2>&1 | tail -2
timeout 300 python bench.py --steps 20 --warmup 5 --no-cpu-baseline --e2e-steps 2 > gpurun_out/bench.json; python -c "import json;d=json.load(open('gpurun_out/bench.json'));print(d['value'],d['breakdown_ms'],d['roofline']['frac'], d['roofline_k1']['frac'])"
timeout 300 python bench.py --config w8a8_4096_m256 --steps 20 --warmup 5 --no-cpu-baseline --e2e-steps 2 > gpurun_out/bench0.json; python -c "import json;d=json.load(open('gpurun_out/bench0.json'));print(d['value'],d['breakdown_ms'],d['roofline']['frac'], d['roofline_k1']['frac'])"
