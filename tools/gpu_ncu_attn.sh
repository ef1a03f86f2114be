nvcc -gencode arch=compute_100a,code=sm_100a -O2 -std=c++20 -lineinfo tools/attn_check.cu -o /tmp/attn_check -L paper_2605_08314_b200 -lfsvd_b200 -Xlinker -rpath=$PWD/paper_2605_08314_b200 || exit 1
mkdir -p gpurun_out/final
# the last (largest) case of attn_check: 4 x 40 heads x 1024 queries at history 1024 -- skip the earlier launches
timeout 900 ncu --set full --import-source on --clock-control none -k regex:attn_tc_kernel -s 8 -c 1 -o gpurun_out/final/prof_attn_big /tmp/attn_check > gpurun_out/final/ncu_attn_big.log 2>&1; echo rc=$?
