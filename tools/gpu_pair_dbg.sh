# k-order stagger (dbg bit 1) and operand-stream-only (bit 0) at the C2 prefill shapes (gemm_sweep: weights > L2)
nvcc -gencode arch=compute_100a,code=sm_100a -O2 -std=c++20 -I include tools/gemm_sweep.cu -o /tmp/gemm_sweep -L paper_2605_08314_b200 -lfsvd_b200 -Xlinker -rpath=$PWD/paper_2605_08314_b200 || exit 1
for d in 0 1 2 3; do
  echo "== dbg=$d"
  FSVD_GEMM_DBG=$d timeout 120 /tmp/gemm_sweep 512 1 pair 2>&1 | grep -E "auto|BN=128 BMT=1 CG=2|BN=256 BMT=1 CG=2|BN=160 BMT=1 CG=2" | sed 's/maxdiff.*//'
done
