for a in 0 8 16 32; do FSVD_MK_L2_AHEAD=$a timeout 300 python bench.py --steps 2 --warmup 2 --no-cpu-baseline --gen 64 2>&1 | tail -1 | python -c "
import json,sys; d=json.loads(sys.stdin.read()); print('l2_ahead', $a, 'decode ms/tok', round(d['decode_ms_per_token'],3), 'frac', round(d['roofline']['frac'],3))"; done
