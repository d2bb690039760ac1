# quick GPU validation: parity tests + headline bench line
timeout 600 python -m pytest tests/test_gpu_parity.py -x -q 2>&1 | tail -5
timeout 300 python bench.py --steps 20 --warmup 5 --no-cpu-baseline --e2e-steps 2 2>&1 | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print(json.dumps({k:d[k] for k in ['value','ms_per_step','breakdown_ms','roofline_k1','clocks']}))"
