# cluster (DSMEM) split-K reduction in the decode-sized swap GEMM: correctness + timing, then C3/C4/C5 with/without
nvcc -gencode arch=compute_100a,code=sm_100a -O2 -std=c++20 -I include tools/gemm_sweep.cu -o /tmp/gemm_sweep -L paper_2605_08314_b200 -lfsvd_b200 -Xlinker -rpath=$PWD/paper_2605_08314_b200 || exit 1
for m in 8 16 32; do timeout 120 /tmp/gemm_sweep $m 8 cred 2>&1 | sed 's/(max|y|.*//'; done > gpurun_out/cred_sweep.log 2>&1
for c in c3 c4 c5; do
  FSVD_NO_CRED=1 timeout 300 python bench.py --config $c --steps 1 --warmup 3 2>/dev/null | tail -1 > gpurun_out/cred_${c}_off.json
  timeout 300 python bench.py --config $c --steps 1 --warmup 3 2>/dev/null | tail -1 > gpurun_out/cred_${c}_on.json
done
