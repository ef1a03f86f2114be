timeout 300 python -m pytest tests/test_gpu_parity.py -x -q > gpurun_out/db_parity.log 2>&1; echo "parity rc=$?"; tail -1 gpurun_out/db_parity.log
timeout 600 python bench.py --steps 3 --warmup 3 --no-c5 --no-cpu-baseline > gpurun_out/db_bench.log 2>&1; echo "bench rc=$?"; grep -o '"decode_ms_per_token": [0-9.]*\|"prefill_ms": [0-9.]*\|"frac": [0-9.]*' gpurun_out/db_bench.log | head -3
