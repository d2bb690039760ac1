timeout 900 python -m pytest tests/test_gpu_epilogue.py tests/test_gpu_full.py tests/test_gpu_parity.py -x -q 2>&1 | tail -3
FQG_GEMM_DEBUG=1 timeout 120 python tools/layer_gemm_dbg.py 2>&1 | grep -E "accumulator ready|per CTA: mma|per leader" | tail -3
timeout 300 python bench.py --steps 20 --warmup 5 --no-cpu-baseline --no-subresults --e2e-steps 2 > gpurun_out/bench.json; python -c "import json;d=json.load(open('gpurun_out/bench.json'));print(d['value'],d['breakdown_ms'],d['roofline']['frac'])"
FQG_GEMM_NB=2 timeout 300 python bench.py --steps 20 --warmup 5 --no-cpu-baseline --no-subresults --e2e-steps 2 > gpurun_out/bench2.json; python -c "import json;d=json.load(open('gpurun_out/bench2.json'));print('NB2', d['value'],d['breakdown_ms'],d['roofline']['frac'])"
