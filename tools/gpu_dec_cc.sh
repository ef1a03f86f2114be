timeout 300 python -m pytest tests/test_gpu_parity.py tests/test_gpu_multistep.py -x -q > gpurun_out/cc_parity.log 2>&1; echo "parity rc=$?"; tail -2 gpurun_out/cc_parity.log
timeout 600 python -m pytest tests/test_gpu_regime.py -x -q -s -k "7b or c1" > gpurun_out/cc_regime.log 2>&1; echo "regime rc=$?"; grep -E "rel err|passed|failed" gpurun_out/cc_regime.log | tail -4
timeout 600 python bench.py --steps 3 --warmup 3 --no-c5 --no-cpu-baseline > gpurun_out/cc_bench.log 2>&1; echo "bench rc=$?"; grep -o '"decode_ms_per_token": [0-9.]*\|"frac": [0-9.]*' gpurun_out/cc_bench.log | head -2
timeout 300 python tools/trace_decode.py > gpurun_out/cc_trace.log 2>&1; grep -A11 "per-CTA phase duration" gpurun_out/cc_trace.log; grep -A12 "^L16.qkvA: staged" gpurun_out/cc_trace.log | head -3
