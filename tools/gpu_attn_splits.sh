# batched decode attention: bulk-copy kernel split sweep vs the register kernel, C3 and C5 shapes
for S in 0 1 2 3 4 6; do
  if [ $S = 0 ]; then E=""; else E="FSVD_ATTN_SPLITS=$S"; fi
  env $E timeout 600 python tools/batched_trace.py 2>&1 | grep -E "step|attn_decode" | head -2 | sed "s/^/C3 S=$S /"
done
FSVD_ATTN_DEC_REG=1 timeout 600 python tools/batched_trace.py 2>&1 | grep -E "step|attn_decode" | head -2 | sed "s/^/C3 reg /"
for S in 0 1 2; do
  if [ $S = 0 ]; then E=""; else E="FSVD_ATTN_SPLITS=$S"; fi
  env $E timeout 600 python tools/batched_trace.py --batch 32 --ctx 1024 --family B 2>&1 | grep -E "step|attn_decode" | head -2 | sed "s/^/C5 S=$S /"
done
FSVD_ATTN_DEC_REG=1 timeout 600 python tools/batched_trace.py --batch 32 --ctx 1024 --family B 2>&1 | grep -E "step|attn_decode" | head -2 | sed "s/^/C5 reg /"
timeout 900 python -m pytest tests/test_gpu_batched.py tests/test_gpu_regime.py -m gpu -x -q 2>&1 | tail -2
