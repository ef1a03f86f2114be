nvcc -gencode arch=compute_100a,code=sm_100a -O2 -std=c++20 -I include tools/gemm_bench.cu -o /tmp/gemm_bench -L paper_2605_08314_b200 -lfsvd_b200 -Xlinker -rpath=$PWD/paper_2605_08314_b200 || exit 1
for shp in "512 3696 4096" "512 4096 1280" "512 1792 11008" "512 4096 4096" "2048 4096 4096" "8192 8192 8192"; do
  for bn in 128 256; do
    for dbg in 0 1; do
      echo -n "BN=$bn nomma=$dbg "; FSVD_GEMM_BN=$bn FSVD_GEMM_DBG=$dbg timeout 60 /tmp/gemm_bench $shp 20 2>&1 | tail -1
    done
  done
done
