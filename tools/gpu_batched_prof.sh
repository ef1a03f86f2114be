# one decode step of the batched engine: launch list + full captures of the swap GEMM (ugB) and flash decode
timeout 900 ncu --set full --clock-control none -k gemm_swap_kernel --launch-skip 4 --launch-count 1 -o gpurun_out/prof_swap_ugB python tools/batched_once.py > gpurun_out/ncu_swap.log 2>&1
ls -la gpurun_out/prof_swap_ugB.ncu-rep gpurun_out/prof_attn_decode.ncu-rep
