timeout 1500 python -m pytest tests/test_gpu_regime.py tests/test_gpu_parity.py tests/test_gpu_multistep.py -m gpu -x -q 2>&1 | tail -2
timeout 600 python bench.py --steps 3 --warmup 3 --no-c5 --no-cpu-baseline 2>/dev/null | tail -1 > gpurun_out/qc.json
python -c "import json; d=json.load(open('gpurun_out/qc.json')); print('decode', round(d['decode_ms_per_token'],4), 'ms/token', round(d['roofline']['frac'],4), 'prefill', round(d['prefill_ms'],3))"
