timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 3000 --csv --log-file gpurun_out/launches.csv python bench.py --steps 1 --warmup 0 --gen 4 --no-cpu-baseline > gpurun_out/ncu_bench.log 2>&1
python - <<'PY'
import csv,collections
rows=list(csv.reader(open('gpurun_out/launches.csv')))
hdr=None; agg=collections.defaultdict(lambda:[0,0.0])
for r in rows:
    if r and r[0]=='ID': hdr=r; continue
    if hdr and len(r)==len(hdr):
        d=dict(zip(hdr,r))
        if d.get('Metric Name')=='gpu__time_duration.sum':
            k=d['Kernel Name'][:80]; agg[k][0]+=1; agg[k][1]+=float(d['Metric Value'])
tot=sum(v[1] for v in agg.values())
for k,v in sorted(agg.items(),key=lambda x:-x[1][1])[:14]: print(f"{v[0]:6d} {v[1]/1e3:10.1f}us {100*v[1]/tot:5.1f}% {k}")
PY
