timeout 600 python -m pytest tests/test_gpu_parity.py -x -q -k "test_accumulators_and_outputs" 2>&1 | grep -E "Error|assert|mismatch|passed|failed" | head -20
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_flatten16 -s 3 -c 1 -o gpurun_out/prof_k1 python bench.py --steps 2 --warmup 3 --no-cpu-baseline --e2e-steps 1 > /dev/null 2>&1
ls gpurun_out
