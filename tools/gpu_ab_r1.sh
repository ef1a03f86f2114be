for v in old new old new; do
  if [ $v = old ]; then B=tools/ab_r1/bench.py; else B=bench.py; fi
  timeout 600 python $B --steps 3 --warmup 3 --no-c5 --no-cpu-baseline > gpurun_out/ab_$v.log 2>&1
  echo "$v $(grep -o '"decode_ms_per_token": [0-9.]*' gpurun_out/ab_$v.log)"
done
