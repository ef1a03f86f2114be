timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; tail -3 gpurun_out/pytest_gpu.log
for E in "X=1" "FSVD_NO_PDL=1"; do
env $E timeout 300 python bench.py --steps 3 --warmup 3 --gen 64 --no-cpu-baseline > gpurun_out/pfenv.log 2>&1
python -c "import json; j=json.loads(open('gpurun_out/pfenv.log').read().strip().splitlines()[-1]); print('$E prefill ms', round(j['prefill_ms'],2), 'TF', round(j['prefill_tflops'],1), 'decode', round(j['decode_ms_per_token'],3))"
done
