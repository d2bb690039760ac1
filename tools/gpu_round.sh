# One GPU evidence round: tests, smoke, bench lines, reference arm, ncu launch
# list + full captures of K1 and K4 (summarised into profiles/ by
# tools/summarize_ncu.py).
set -x
mkdir -p gpurun_out
nproc
timeout 900 python -m pytest tests -x -q -m gpu > gpurun_out/pytest_gpu.log 2>&1; tail -3 gpurun_out/pytest_gpu.log
timeout 120 python -c "import __graft_entry__ as g; g.smoke()"
timeout 300 python bench.py --steps 20 --warmup 5 > gpurun_out/bench_a8.json 2> gpurun_out/bench_a8.err; cat gpurun_out/bench_a8.json; tail -3 gpurun_out/bench_a8.err
timeout 300 python bench.py --a-format i4 --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/bench_a4.json; cat gpurun_out/bench_a4.json
timeout 300 python bench.py --b-format i8 --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/bench_w8store.json; cat gpurun_out/bench_w8store.json
timeout 300 python bench.py --config w8a8_4096_m256 --steps 20 --warmup 5 > gpurun_out/bench_w8.json; cat gpurun_out/bench_w8.json
timeout 300 python bench.py --config sweep_8192 --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/bench_8192.json; cat gpurun_out/bench_8192.json
timeout 300 python bench.py --config llama13b_up --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/bench_llama.json; cat gpurun_out/bench_llama.json
timeout 300 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/bench_ref.json; cat gpurun_out/bench_ref.json
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -c 40 --csv --log-file gpurun_out/launches.csv python bench.py --steps 3 --warmup 3 --no-cpu-baseline --e2e-steps 1 > /dev/null
timeout 400 ncu --set full --clock-control none --import-source on -k regex:k_gemm_i8 -s 3 -c 1 -o gpurun_out/prof_gemm python bench.py --steps 2 --warmup 3 --no-cpu-baseline --e2e-steps 1 > /dev/null
timeout 400 ncu --set full --clock-control none --import-source on -k regex:k_flatten -s 3 -c 1 -o gpurun_out/prof_k1 python bench.py --steps 2 --warmup 3 --no-cpu-baseline --e2e-steps 1 > /dev/null
ls -la gpurun_out
