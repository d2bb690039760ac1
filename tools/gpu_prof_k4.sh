set -x
mkdir -p gpurun_out
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_gemm_i8_pair -s 2 -c 1 -o gpurun_out/prof_k4 python tools/layer_gemm_dbg.py > /dev/null 2>&1
ls -la gpurun_out
