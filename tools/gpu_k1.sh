#!/bin/bash
# K1 A/B on the GPU box: parity tests, then the layer breakdown (optionally per rows-per-block).
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_k1_fast.py tests/test_gpu_full.py tests/test_gpu_parity.py -m gpu -x -q > gpurun_out/k1_t.log 2>&1
tail -3 gpurun_out/k1_t.log
for cfg in w4a4_4096 w8a8_4096_m256; do
  for r in ${K1_ROWS:-0}; do
    if [ "$r" = 0 ]; then unset FQG_K1_ROWS; else export FQG_K1_ROWS=$r; fi
    timeout 200 python bench.py --config $cfg --no-subresults --no-cpu-baseline > gpurun_out/k1_b.log 2>&1
    echo "$cfg R=$r $(grep -o '"breakdown_ms[^}]*}' gpurun_out/k1_b.log)"
  done
done
unset FQG_K1_ROWS
if [ -n "$K1_NCU" ]; then
  timeout 300 ncu --set full --import-source on -k regex:k_flatten16 -c 1 -o gpurun_out/prof_k1 -f \
    python bench.py --config w4a4_4096 --no-subresults --no-cpu-baseline --steps 3 --warmup 3 > gpurun_out/k1_ncu.log 2>&1
  tail -2 gpurun_out/k1_ncu.log
fi
