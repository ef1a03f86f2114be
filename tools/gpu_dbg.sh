python tools/dbg_tiny.py 2>&1 | grep -v nonzero > gpurun_out/dbg.log 2>&1
timeout 600 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; tail -3 gpurun_out/pytest_gpu.log
timeout 300 python tools/trace_decode.py > gpurun_out/trace_v2.log 2>&1; head -16 gpurun_out/trace_v2.log
timeout 300 python bench.py --steps 2 --warmup 2 --no-cpu-baseline 2>&1 | tail -1 | python -c "
import json,sys; d=json.loads(sys.stdin.read()); print('decode ms/tok', round(d['decode_ms_per_token'],3), 'frac', round(d['roofline']['frac'],3), 'prefill ms', round(d['prefill_ms'],2))"
