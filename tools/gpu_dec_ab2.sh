# decode A/B with parity guard: toy parity + multistep, then bench decode + trace
timeout 300 python -m pytest tests/test_gpu_parity.py tests/test_gpu_multistep.py -x -q > gpurun_out/ab_parity.log 2>&1; echo "parity rc=$?"; tail -2 gpurun_out/ab_parity.log
timeout 600 python bench.py --steps 3 --warmup 3 --no-c5 --no-cpu-baseline > gpurun_out/ab_bench.log 2>&1; echo "bench rc=$?"; grep -o '"decode_ms_per_token": [0-9.]*\|"prefill_ms": [0-9.]*\|"frac": [0-9.]*' gpurun_out/ab_bench.log | head -3
timeout 300 python tools/trace_decode.py > gpurun_out/ab_trace.log 2>&1; grep -A11 "per-CTA phase duration" gpurun_out/ab_trace.log; grep "step total" gpurun_out/ab_trace.log
