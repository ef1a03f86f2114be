# short tail chunks in the decode megakernel: A/B on one box
for t in "0,3" "24,3" "16,4" "32,4" "33,3" "44,4"; do
  FSVD_MK_TAIL=$t timeout 600 python bench.py --steps 5 --warmup 3 --no-c5 2>/dev/null | tail -1 > gpurun_out/bt.json
  python -c "import json; d=json.load(open('gpurun_out/bt.json')); print('tail=$t', round(d['ms_per_step']/256, 4), 'ms/token', round(d['roofline']['frac'],4))"
done
