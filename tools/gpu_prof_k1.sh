# ncu --set full capture of the K1 kernel (bench workload), source-correlated.
mkdir -p gpurun_out
timeout 400 ncu --set full --clock-control none --import-source on -k regex:k_flatten -s 3 -c 1 -o gpurun_out/prof_k1 python bench.py --steps 2 --warmup 3 --no-cpu-baseline --e2e-steps 1 > /dev/null 2>&1
ls -la gpurun_out
