nvcc -gencode arch=compute_100a,code=sm_100a -O2 -std=c++20 -I include tools/gemm_sweep.cu -o /tmp/gemm_sweep -L paper_2605_08314_b200 -lfsvd_b200 -Xlinker -rpath=$PWD/paper_2605_08314_b200 || exit 1
timeout 300 /tmp/gemm_sweep 512 4 cred512 > gpurun_out/cred512.log 2>&1; echo "rc=$?" >> gpurun_out/cred512.log
