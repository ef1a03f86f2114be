# round 2: new regime parity tests + full GPU suite + bench (with C5 leg) + reference arm
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
nproc
timeout 1500 python -m pytest tests -m gpu -x -q -s -k "regime" > gpurun_out/pytest_regime.log 2>&1; tail -15 gpurun_out/pytest_regime.log
timeout 900 python -m pytest tests -m gpu -x -q -k "not regime" > gpurun_out/pytest_gpu.log 2>&1; tail -3 gpurun_out/pytest_gpu.log
timeout 900 python bench.py --steps 3 --warmup 3 > gpurun_out/bench.log 2>&1; tail -1 gpurun_out/bench.log
timeout 600 python bench.py --impl reference --steps 5 --warmup 2 > gpurun_out/ref.log 2>&1; tail -1 gpurun_out/ref.log
