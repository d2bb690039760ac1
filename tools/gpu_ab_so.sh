#!/bin/bash
# A/B of two builds of libfqg.so (the tree's and abtmp/libfqg_b.so) on one box, alternating.
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
cp paper_2402_17985_b200/libfqg.so abtmp/libfqg_a.so
for rep in 1 2; do
  for v in a b; do
    cp abtmp/libfqg_$v.so paper_2402_17985_b200/libfqg.so
    for cfg in ${AB_CONFIGS:-w8a8_4096_m256}; do
      timeout 200 python bench.py --config $cfg --no-subresults --no-cpu-baseline > gpurun_out/ab.log 2>&1
      echo "$v $cfg $(grep -o '"breakdown_ms[^}]*}' gpurun_out/ab.log)"
    done
  done
done
cp abtmp/libfqg_a.so paper_2402_17985_b200/libfqg.so
