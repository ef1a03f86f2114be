nvcc -gencode arch=compute_100a,code=sm_100a -O2 -std=c++20 -I include tools/gemm_sweep.cu -o /tmp/gemm_sweep -L paper_2605_08314_b200 -lfsvd_b200 -Xlinker -rpath=$PWD/paper_2605_08314_b200 || exit 1
if [ "$2" = "san" ]; then
  FSVD_GEMM_BN=128 FSVD_GEMM_CG=2 timeout 300 compute-sanitizer --tool memcheck /tmp/gemm_sweep 512 1 pair oB > gpurun_out/pair_san.log 2>&1; echo "rc=$?" >> gpurun_out/pair_san.log
  head -60 gpurun_out/pair_san.log
fi
timeout 120 /tmp/gemm_sweep 512 ${1:-3} pair > gpurun_out/pair512.log 2>&1; echo "rc=$?" >> gpurun_out/pair512.log
tail -5 gpurun_out/pair512.log
