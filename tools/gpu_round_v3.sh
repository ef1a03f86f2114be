nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 600 python bench.py --steps 3 --warmup 3 > gpurun_out/bench_v3.log 2>&1; tail -1 gpurun_out/bench_v3.log | cut -c1-400
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 3000 --csv --log-file gpurun_out/launches_v3.csv python bench.py --steps 1 --warmup 0 --gen 8 --no-cpu-baseline > gpurun_out/ncu_bench_v3.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:decode_mk -s 2 -c 1 -o gpurun_out/prof_step32_v3 python tools/mk_profile_run.py 32 > gpurun_out/ncu_step_v3.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:gemm_tc_kernel --launch-skip 261 --launch-count 1 -o gpurun_out/prof_ugB_v3 python tools/prefill_once.py > gpurun_out/ncu_ugB_v3.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:gemm_tc_kernel --launch-skip 256 --launch-count 1 -o gpurun_out/prof_qkvA_v3 python tools/prefill_once.py > gpurun_out/ncu_qkvA_v3.log 2>&1
ls -la gpurun_out/*v3*
