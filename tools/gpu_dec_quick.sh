timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; tail -2 gpurun_out/pytest_gpu.log
timeout 300 python bench.py --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/dq.log 2>&1
python -c "import json; j=json.loads(open('gpurun_out/dq.log').read().strip().splitlines()[-1]); print('decode', round(j['decode_ms_per_token'],4), round(j['roofline']['frac'],4), 'prefill', round(j['prefill_ms'],2), j['engine'])"
