#!/bin/bash
# K4 tile-shape A/B at the headline: B format x FQG_GEMM_NB.
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
for bf in i4 i8; do
  for nb in 0 1; do
    if [ "$nb" = 0 ]; then unset FQG_GEMM_NB; else export FQG_GEMM_NB=$nb; fi
    timeout 200 python bench.py --config w4a4_4096 --b-format $bf --no-subresults --no-cpu-baseline > gpurun_out/nb_b.log 2>&1
    echo "b=$bf NB=$nb $(grep -o '"breakdown_ms[^}]*}' gpurun_out/nb_b.log)"
  done
done
export FQG_GEMM_NB=1
for bf in 6 5; do
  FQG_GEMM_DEBUG=1 timeout 120 python tools/layer_gemm_dbg.py $bf > gpurun_out/nb_dbg_$bf.txt 2>&1
  head -4 gpurun_out/nb_dbg_$bf.txt
done
