# same-box A/B of builds of libfsvd_b200.so under ab/ (decode bench, alternating); args: names
for round in 1 2; do
for v in "$@"; do
  cp ab/$v.so paper_2605_08314_b200/libfsvd_b200.so
  timeout 600 python bench.py --steps 5 --warmup 3 --no-c5 2>/dev/null | tail -1 > gpurun_out/ab_$v.json
  python -c "import json; d=json.load(open('gpurun_out/ab_$v.json')); print('$v', round(d['ms_per_step']/256, 4), 'ms/token', round(d['roofline']['frac'],4), 'prefill', round(d['prefill_ms'],3))"
done
done
