nvcc -gencode arch=compute_100a,code=sm_100a -O2 -std=c++20 tools/attn_check.cu -o /tmp/attn_check -L paper_2605_08314_b200 -lfsvd_b200 -Xlinker -rpath=$PWD/paper_2605_08314_b200 || exit 1
timeout 300 /tmp/attn_check > gpurun_out/attn_check.log 2>&1; echo "rc=$?" >> gpurun_out/attn_check.log
cat gpurun_out/attn_check.log
python tools/pf_trace.py --label fa4 2>&1 | grep "prefill 512"
FSVD_ATTN_MMA=1 python tools/pf_trace.py --label mma 2>&1 | grep "prefill 512"
