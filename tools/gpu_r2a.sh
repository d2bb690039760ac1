# Round-2 baseline: GPU suite, bench, K4 phase debug, ncu full capture of K4 with source.
set -x
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 900 python -m pytest tests -x -q -m gpu > gpurun_out/pytest_gpu.log 2>&1; tail -3 gpurun_out/pytest_gpu.log
timeout 300 python bench.py --steps 20 --warmup 5 --no-cpu-baseline --e2e-steps 2 > gpurun_out/bench.json; cat gpurun_out/bench.json
FQG_GEMM_DEBUG=1 timeout 120 python tools/gemm_once.py 2048 4096 7488 5 6 2> gpurun_out/gemm_dbg_i4.txt; tail -12 gpurun_out/gemm_dbg_i4.txt
FQG_GEMM_DEBUG=1 timeout 120 python tools/gemm_once.py 2048 4096 7488 5 5 2> gpurun_out/gemm_dbg_i8.txt; tail -12 gpurun_out/gemm_dbg_i8.txt
timeout 300 python tools/gemm_sweep.py > gpurun_out/sweep.txt 2>&1; cat gpurun_out/sweep.txt
timeout 400 ncu --set full --clock-control none --import-source on -k regex:k_gemm_i8 -s 3 -c 1 -o gpurun_out/prof_gemm python bench.py --steps 2 --warmup 3 --no-cpu-baseline --e2e-steps 1 > /dev/null 2>&1
ls -la gpurun_out
