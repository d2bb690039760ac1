# Quick GPU iteration: new/focused tests, full GPU suite, one bench line.
set -x
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_k1_fast.py -x -q 2>&1 | tail -15
timeout 900 python -m pytest tests -x -q -m gpu 2>&1 | tail -5
timeout 300 python bench.py --steps 20 --warmup 5 --no-cpu-baseline --e2e-steps 2 > gpurun_out/bench_q.json; cat gpurun_out/bench_q.json
timeout 300 python bench.py --a-format i4 --steps 20 --warmup 5 --no-cpu-baseline --e2e-steps 2 > gpurun_out/bench_q4.json; cat gpurun_out/bench_q4.json
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -c 12 --csv --log-file gpurun_out/launches_q.csv python bench.py --steps 3 --warmup 3 --no-cpu-baseline --e2e-steps 1 > /dev/null
