timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; tail -2 gpurun_out/pytest_gpu.log
timeout 600 python bench.py --steps 3 --warmup 3 > gpurun_out/bench.log 2>&1; tail -1 gpurun_out/bench.log | python -c "
import json,sys; d=json.loads(sys.stdin.read()); print('decode ms/tok', round(d['decode_ms_per_token'],3), 'tok/s', round(d['value'],1), 'frac', round(d['roofline']['frac'],3), 'prefill ms', round(d['prefill_ms'],2), 'e2e', round(d['e2e']['value'],1), 'cpu', d['cpu_baseline'])"
