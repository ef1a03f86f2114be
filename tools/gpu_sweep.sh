nvcc -gencode arch=compute_100a,code=sm_100a -O2 -std=c++20 -I include tools/gemm_sweep.cu -o /tmp/gemm_sweep -L paper_2605_08314_b200 -lfsvd_b200 -Xlinker -rpath=$PWD/paper_2605_08314_b200 || exit 1
timeout 300 /tmp/gemm_sweep 512 > gpurun_out/sweep512.log 2>&1
timeout 300 /tmp/gemm_sweep 2048 > gpurun_out/sweep2048.log 2>&1
timeout 300 /tmp/gemm_sweep 16 > gpurun_out/sweep16.log 2>&1
