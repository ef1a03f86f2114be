timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; tail -3 gpurun_out/pytest_gpu.log
timeout 300 python bench.py --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/bench.log 2>&1
python -c "import json; j=json.loads(open('gpurun_out/bench.log').read().strip().splitlines()[-1]); print('decode', round(j['decode_ms_per_token'],4), round(j['roofline']['frac'],4), 'prefill', j['prefill_ms'])"
timeout 300 python tools/trace_decode.py > gpurun_out/trace.log 2>&1; sed -n 2,16p gpurun_out/trace.log; grep -A12 "per-CTA phase" gpurun_out/trace.log
