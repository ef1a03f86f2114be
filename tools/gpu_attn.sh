# GPU tests, C2 prefill time, and the prefill attention kernel's time per layer (ncu launch list)
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; tail -2 gpurun_out/pytest_gpu.log
timeout 300 python bench.py --steps 3 --warmup 3 --gen 64 --no-cpu-baseline > gpurun_out/pfenv.log 2>&1
python -c "import json; j=json.loads(open('gpurun_out/pfenv.log').read().strip().splitlines()[-1]); print('prefill ms', round(j['prefill_ms'],3), 'TF', round(j['prefill_tflops'],1))"
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"attn_prefill" --csv --log-file gpurun_out/attn.csv python tools/prefill_once.py > /dev/null 2>&1
python -c "
import csv
r=list(csv.reader(open('gpurun_out/attn.csv'))); hi=[i for i,x in enumerate(r) if 'Kernel Name' in x][0]; h=r[hi]; v=h.index('Metric Value')
t=[float(x[v].replace(',','')) for x in r[hi+1:] if len(x)>v]; print('attn per layer us', sum(t[len(t)//2:])/len(t[len(t)//2:])/1e3)"
