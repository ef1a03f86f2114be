timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; tail -2 gpurun_out/pytest_gpu.log
for E in "FSVD_MK_EXACT=1" "FSVD_MK_EXACT=0"; do
env $E timeout 300 python bench.py --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/ex.log 2>&1
python -c "import json; j=json.loads(open('gpurun_out/ex.log').read().strip().splitlines()[-1]); print('$E decode', round(j['decode_ms_per_token'],4), round(j['roofline']['frac'],4))"
done
FSVD_MK_EXACT=1 timeout 300 python tools/trace_decode.py > gpurun_out/trace.log 2>&1; grep -A11 "per-CTA phase" gpurun_out/trace.log
