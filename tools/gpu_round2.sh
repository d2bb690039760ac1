# Round-2 evidence: GPU suite, smoke, bench (N=1, with subresults), reference arm,
# ncu launch list of the bench step, full captures of K1 and K4 (headline workload).
set -x
mkdir -p gpurun_out
nproc
timeout 1500 python -m pytest tests -x -q -m gpu > gpurun_out/pytest_gpu.log 2>&1; tail -3 gpurun_out/pytest_gpu.log
timeout 120 python -c "import __graft_entry__ as g; g.smoke()"
timeout 600 python bench.py --steps 20 --warmup 5 > gpurun_out/bench_main.json 2> gpurun_out/bench_main.err; tail -c 600 gpurun_out/bench_main.json; tail -3 gpurun_out/bench_main.err
timeout 300 python bench.py --a-format i4 --steps 20 --warmup 5 --no-cpu-baseline --no-subresults > gpurun_out/bench_a4.json
timeout 300 python bench.py --b-format i8 --steps 20 --warmup 5 --no-cpu-baseline --no-subresults > gpurun_out/bench_w8store.json
timeout 300 python bench.py --config w8a8_4096_m256 --steps 20 --warmup 5 --no-subresults > gpurun_out/bench_cfg0.json
timeout 300 python bench.py --config llama13b_up --steps 10 --warmup 3 --no-cpu-baseline --no-subresults > gpurun_out/bench_llama.json
timeout 300 python bench.py --config sweep_8192 --steps 10 --warmup 3 --no-cpu-baseline --no-subresults > gpurun_out/bench_8192.json
timeout 300 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/bench_ref.json; cat gpurun_out/bench_ref.json | cut -c1-300
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 60 --csv --log-file gpurun_out/launches.csv python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-subresults --e2e-steps 1 > /dev/null 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_gemm_i8_pair -s 3 -c 1 -o gpurun_out/prof_gemm python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-subresults --e2e-steps 1 > /dev/null 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_flatten16 -s 3 -c 1 -o gpurun_out/prof_k1 python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-subresults --e2e-steps 1 > /dev/null 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_gemm_i8_pair -s 3 -c 1 -o gpurun_out/prof_gemm_m256 python bench.py --config w8a8_4096_m256 --steps 2 --warmup 3 --no-cpu-baseline --no-subresults --e2e-steps 1 > /dev/null 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 60 --csv --log-file gpurun_out/launches_m256.csv python bench.py --config w8a8_4096_m256 --steps 3 --warmup 3 --no-cpu-baseline --no-subresults --e2e-steps 1 > /dev/null 2>&1
ls -la gpurun_out
