#!/bin/bash
# K1 CTA size x rows-per-block A/B (FQG_K1_THREADS / FQG_K1_ROWS), parity first.
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
FQG_K1_THREADS=128 timeout 600 python -m pytest tests/test_gpu_k1_fast.py tests/test_gpu_full.py -m gpu -x -q > gpurun_out/k1t_t.log 2>&1
tail -1 gpurun_out/k1t_t.log
for cfg in w4a4_4096 w8a8_4096_m256; do
  for t in 256 128; do
    for r in ${K1_ROWS:-0}; do
      if [ "$r" = 0 ]; then unset FQG_K1_ROWS; else export FQG_K1_ROWS=$r; fi
      FQG_K1_THREADS=$t timeout 200 python bench.py --config $cfg --no-subresults --no-cpu-baseline > gpurun_out/k1t_b.log 2>&1
      echo "$cfg T=$t R=$r $(grep -o '"flatten_quant_K1": [0-9.]*' gpurun_out/k1t_b.log) $(grep -o '"K1_K4_graph": [0-9.]*' gpurun_out/k1t_b.log)"
    done
  done
done
