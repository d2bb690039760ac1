mkdir -p gpurun_out
FQG_GEMM_VARIANT=2 timeout 300 ncu --set full --clock-control none --import-source on -k regex:k_gemm -s 2 -c 1 -o gpurun_out/prof_gemm_pair python tools/gemm_once.py 2048 4096 7296 > /dev/null 2>&1
FQG_GEMM_VARIANT=1 timeout 300 ncu --set full --clock-control none --import-source on -k regex:k_gemm -s 2 -c 1 -o gpurun_out/prof_gemm_one python tools/gemm_once.py 2048 4096 7296 > /dev/null 2>&1
ls -la gpurun_out/*.ncu-rep
