timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; tail -2 gpurun_out/pytest_gpu.log
for c in c3 c4 c5; do
timeout 900 python bench.py --config $c --steps 1 --warmup 3 --no-cpu-baseline > gpurun_out/cfg_$c.log 2>&1
python -c "import json; j=json.loads(open('gpurun_out/cfg_$c.log').read().strip().splitlines()[-1]); print('$c tok/s', round(j['value'],1), 'ms/step', round(j['decode_ms_per_token'],3), 'frac', round(j['roofline']['frac'],3), 'prefill ms', round(j['prefill_ms'],1), 'TF', round(j['prefill_tflops'],1), 'e2e', round(j['e2e']['value'],1))"
done
