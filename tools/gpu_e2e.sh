timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; tail -2 gpurun_out/pytest_gpu.log
timeout 300 python bench.py --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/e2e.log 2>&1
python -c "import json; j=json.loads(open('gpurun_out/e2e.log').read().strip().splitlines()[-1]); print('decode', round(j['decode_ms_per_token'],4), 'tok/s', round(j['value'],1), 'e2e', round(j['e2e']['value'],1), 'prefill', round(j['prefill_ms'],2))"
