timeout 300 python -m pytest tests/test_gpu_parity.py -x -q > gpurun_out/q_parity.log 2>&1; echo "parity rc=$?"; tail -1 gpurun_out/q_parity.log
timeout 600 python bench.py --steps 3 --warmup 3 --no-c5 --no-cpu-baseline > gpurun_out/q_bench.log 2>&1; echo "bench rc=$?"; grep -o '"decode_ms_per_token": [0-9.]*\|"frac": [0-9.]*' gpurun_out/q_bench.log | head -2
timeout 300 python tools/trace_decode.py > gpurun_out/q_trace.log 2>&1; grep -A10 "per-CTA phase duration" gpurun_out/q_trace.log; grep -A12 "^L16.qkvA: staged" gpurun_out/q_trace.log | head -2
