nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu_final.log 2>&1; tail -2 gpurun_out/pytest_gpu_final.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()"
timeout 600 python bench.py --steps 3 --warmup 3 > gpurun_out/bench_final.log 2>&1; tail -1 gpurun_out/bench_final.log | cut -c1-300
timeout 600 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/ref_final.log 2>&1; tail -1 gpurun_out/ref_final.log | cut -c1-200
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 3000 --csv --log-file gpurun_out/launches_final.csv python bench.py --steps 1 --warmup 0 --gen 8 --no-cpu-baseline > gpurun_out/ncu_bench_final.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:decode_mk -s 2 -c 1 -o gpurun_out/prof_step32_final python tools/mk_profile_run.py 32 > gpurun_out/ncu_step_final.log 2>&1
ls -la gpurun_out/*final*
