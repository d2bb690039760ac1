timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_flatten16 -s 3 -c 1 -o gpurun_out/prof_k1 python bench.py --steps 2 --warmup 3 --no-cpu-baseline --e2e-steps 1 > /dev/null 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_flatten16 -s 3 -c 1 -o gpurun_out/prof_k1_m256 python bench.py --config w8a8_4096_m256 --steps 2 --warmup 3 --no-cpu-baseline --e2e-steps 1 > /dev/null 2>&1
ls gpurun_out
