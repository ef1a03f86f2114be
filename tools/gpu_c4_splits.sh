# C4-shaped batched decode (13B, family D, B=16, ctx 2560): attention split choice
for S in 0 1 2 3 4; do
  if [ $S = 0 ]; then E=""; else E="FSVD_ATTN_SPLITS=$S"; fi
  env $E timeout 900 python tools/batched_trace.py --preset llama13b --family D --batch 16 --ctx 2560 2>&1 | grep -E "step|attn_decode_bulk" | head -2 | sed "s/^/C4 S=$S /"
done
timeout 600 python tools/batched_trace.py 2>&1 | grep -E "step" | sed "s/^/C3 auto /"
timeout 600 python tools/batched_trace.py --batch 32 --ctx 1024 --family B 2>&1 | grep -E "step" | sed "s/^/C5 auto /"
