# ncu --set full of one layer's prefill GEMMs (second prefill, layer 0: qkvA qkvB oA oB ugA ugB dA dB)
mkdir -p gpurun_out/final
timeout 1200 ncu --set full --clock-control none -k regex:gemm_tc_kernel -s 256 -c 8 -o gpurun_out/final/prof_prefill_gemms python tools/prefill_once.py > gpurun_out/final/ncu_prefill.log 2>&1; echo "rc=$?"
timeout 600 ncu --set full --clock-control none -k regex:attn_tc -s 32 -c 1 -o gpurun_out/final/prof_prefill_attn python tools/prefill_once.py >> gpurun_out/final/ncu_prefill.log 2>&1; echo "rc=$?"
