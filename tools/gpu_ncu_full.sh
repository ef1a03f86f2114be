nvcc -gencode arch=compute_100a,code=sm_100a -O2 -std=c++20 -I include tools/gemm_bench.cu -o /tmp/gemm_bench -L paper_2605_08314_b200 -lfsvd_b200 -Xlinker -rpath=$PWD/paper_2605_08314_b200
timeout 600 ncu --set full --clock-control none --import-source on -k regex:decode_mk -s 2 -c 1 -o gpurun_out/prof_decode python tools/mk_profile_run.py 4 > gpurun_out/ncu1.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:gemm_tc -s 3 -c 1 -o gpurun_out/prof_gemm512 /tmp/gemm_bench 512 4096 4096 2 > gpurun_out/ncu2.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:gemm_tc -s 3 -c 1 -o gpurun_out/prof_gemm8k /tmp/gemm_bench 8192 8192 8192 2 > gpurun_out/ncu3.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:attn_prefill_tc -s 2 -c 1 -o gpurun_out/prof_attn python bench.py --steps 1 --warmup 0 --gen 2 --no-cpu-baseline > gpurun_out/ncu4.log 2>&1
ls -la gpurun_out/*.ncu-rep
