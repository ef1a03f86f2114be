# one ncu --set full capture of the qkvA prefill GEMM (auto config, then the CTA-pair BN=128 config)
nvcc -gencode arch=compute_100a,code=sm_100a -O2 -std=c++20 -I include tools/gemm_sweep.cu -o /tmp/gemm_sweep -L paper_2605_08314_b200 -lfsvd_b200 -Xlinker -rpath=$PWD/paper_2605_08314_b200 || exit 1
timeout 600 ncu --set full --clock-control none -k regex:gemm_tc_kernel -s 2 -c 1 -o gpurun_out/ncu_qkvA_auto /tmp/gemm_sweep 512 1 pair qkvA > gpurun_out/ncu_qkvA.log 2>&1
nvcc -gencode arch=compute_100a,code=sm_100a -O2 -std=c++20 -I include tools/gemm_bench.cu -o /tmp/gemm_bench -L paper_2605_08314_b200 -lfsvd_b200 -Xlinker -rpath=$PWD/paper_2605_08314_b200
FSVD_GEMM_BN=256 FSVD_GEMM_BMT=2 FSVD_GEMM_CG=2 timeout 600 ncu --set full --clock-control none -k regex:gemm_tc_kernel -s 2 -c 1 -o gpurun_out/ncu_2048_pair /tmp/gemm_bench 2048 4096 4096 3 >> gpurun_out/ncu_qkvA.log 2>&1
tail -3 gpurun_out/ncu_qkvA.log
