timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; tail -2 gpurun_out/pytest_gpu.log
timeout 300 python bench.py --steps 3 --warmup 3 --gen 64 --no-cpu-baseline > gpurun_out/pfenv.log 2>&1
python -c "import json; j=json.loads(open('gpurun_out/pfenv.log').read().strip().splitlines()[-1]); print('c2 prefill ms', round(j['prefill_ms'],2), 'TF', round(j['prefill_tflops'],1), 'decode', round(j['decode_ms_per_token'],3))"
for c in c3; do
timeout 600 python bench.py --config $c --steps 1 --warmup 3 --gen 64 --no-cpu-baseline > gpurun_out/pf_$c.log 2>&1
python -c "import json; j=json.loads(open('gpurun_out/pf_$c.log').read().strip().splitlines()[-1]); print('$c prefill ms', round(j['prefill_ms'],2), 'TF', round(j['prefill_tflops'],1), 'decode', round(j['decode_ms_per_token'],3))"
done
