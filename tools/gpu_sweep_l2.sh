# decode megakernel: L2 prefetch distance (chunks beyond the ring) sweep, same box
for D in 5 0 10 16 24 40; do
  FSVD_MK_L2_AHEAD=$D timeout 600 python bench.py --steps 5 --warmup 3 --no-c5 2>/dev/null | tail -1 > gpurun_out/bl2.json
  python -c "import json; d=json.load(open('gpurun_out/bl2.json')); print('D=$D', round(d['ms_per_step']/256, 4), 'ms/token', round(d['roofline']['frac'],4))"
done
