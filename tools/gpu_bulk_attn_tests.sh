timeout 1500 python -m pytest tests -m gpu -x -q 2>&1 | tail -3
for c in c3 c5; do
  timeout 900 python bench.py --config $c --steps 1 --warmup 3 2>/dev/null | tail -1 > gpurun_out/bulk_$c.json
  python -c "import json; d=json.load(open('gpurun_out/bulk_$c.json')); print('$c', round(d['value'],1), d['unit'], 'frac', round(d['roofline']['frac'],4))"
done
