set -x
FSVD_BATCHED=1 timeout 300 python bench.py --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/cfg_c2_batched.log 2>&1; tail -1 gpurun_out/cfg_c2_batched.log | cut -c1-900
timeout 600 python bench.py --config c3 --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/cfg_c3.log 2>&1; tail -1 gpurun_out/cfg_c3.log | cut -c1-1200
timeout 600 python bench.py --config c5 --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/cfg_c5.log 2>&1; tail -1 gpurun_out/cfg_c5.log | cut -c1-1200
timeout 900 python bench.py --config c4 --steps 1 --warmup 1 --no-cpu-baseline > gpurun_out/cfg_c4.log 2>&1; tail -1 gpurun_out/cfg_c4.log | cut -c1-1200
