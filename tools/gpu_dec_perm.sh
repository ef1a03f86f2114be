# permuted decode planes: parity suite + decode timing
timeout 1500 python -m pytest tests -m gpu -x -q 2>&1 | tail -3
timeout 600 python bench.py --steps 5 --warmup 3 --no-c5 2>/dev/null | tail -1 > gpurun_out/bench_perm.json
python - <<'P'
import json; d=json.load(open("gpurun_out/bench_perm.json"))
print("value", d["value"], d["unit"], "ms/step", d["ms_per_step"], "frac", d["roofline"]["frac"], "prefill", d.get("prefill_ms"))
P
