bash tools/gpu_gemm.sh
bash tools/gpu_check.sh
