"""Collect the round's final evidence run (tools/gpu_final_r2.sh, outputs in
gpurun_out/final/) into profiles/: bench lines, the ncu launch list of the bench
command with per-kernel shares, the ncu --set full numbers of the full-step decode
megakernel (-> profiles/traffic.json, which bench.py reports as roofline.traffic)."""
import csv
import collections
import json
import re
import subprocess
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
SRC = ROOT / "gpurun_out" / "final"
TAG = sys.argv[1] if len(sys.argv) > 1 else "r2_final"
OUT = ROOT / "profiles"


def last_json(p):
    for line in reversed(p.read_text().splitlines()):
        line = line.strip()
        if line.startswith("{"):
            return json.loads(line)
    return None


lines = []
for name in ["bench", "ref", "bench_c3", "bench_c4", "bench_c5"]:
    f = SRC / f"{name}.log"
    if f.exists():
        j = last_json(f)
        if j:
            lines.append(j)
(OUT / f"{TAG}_bench.jsonl").write_text("".join(json.dumps(j) + "\n" for j in lines))
print(f"{len(lines)} bench lines -> profiles/{TAG}_bench.jsonl")

# launch list: per-kernel totals over the bench command
lf = SRC / "launches_bench.csv"
if lf.exists():
    rows = list(csv.reader(lf.read_text().splitlines()))
    hi = [i for i, r in enumerate(rows) if "Kernel Name" in r][0]
    h = rows[hi]
    ki, vi, mi = h.index("Kernel Name"), h.index("Metric Value"), h.index("Metric Name")
    agg = collections.OrderedDict()
    for r in rows[hi + 1:]:
        if len(r) > vi and r[mi] == "gpu__time_duration.sum":
            n = re.sub(r"\(.*", "", r[ki].replace("(anonymous namespace)::", ""))[:70]
            a = agg.setdefault(n, [0, 0.0])
            a[0] += 1
            a[1] += float(r[vi].replace(",", ""))
    tot = sum(v[1] for v in agg.values())
    with open(OUT / f"{TAG}_launches_summary.txt", "w") as f:
        f.write(f"ncu launch list of `python bench.py --steps 1 --warmup 3 --gen 8 --no-cpu-baseline --no-c5` "
                f"(serialized, cold caches; shares, not absolute times)\n")
        f.write(f"{'launches':>8} {'total ms':>10} {'share':>7}  kernel\n")
        for n, (c, t) in sorted(agg.items(), key=lambda kv: -kv[1][1]):
            f.write(f"{c:8d} {t / 1e6:10.3f} {100 * t / tot:6.1f}%  {n}\n")
    (OUT / f"{TAG}_launches_bench.csv").write_text(lf.read_text())
    print(f"launch list: {sum(v[0] for v in agg.values())} launches, {len(agg)} kernels")

# ncu --set full of one full-step decode launch
rep = SRC / "prof_step32.ncu-rep"
if rep.exists():
    raw = subprocess.run(["ncu", "-i", str(rep), "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rr = list(csv.reader(raw.splitlines()))
    hdr, units, val = rr[0], rr[1], rr[2]
    m = {hdr[i]: (val[i], units[i]) for i in range(len(hdr))}

    def num(k, scale=1.0):
        v, u = m[k]
        x = float(v.replace(",", ""))
        mult = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "ns": 1e-9, "usecond": 1e-6, "msecond": 1e-3,
                "us": 1e-6, "ms": 1e-3}.get(u, 1.0)
        return x * mult * scale

    rd, wr = num("dram__bytes_read.sum"), num("dram__bytes_write.sum")
    dur = num("gpu__time_duration.sum")
    pct = float(m["dram__bytes_read.sum.pct_of_peak_sustained_elapsed"][0]) + float(
        m["dram__bytes_write.sum.pct_of_peak_sustained_elapsed"][0])
    t = {"decode_step_dram_bytes": rd + wr, "dram_read": rd, "dram_write": wr, "ncu_time_ms": dur * 1e3,
         "dram_pct_of_peak": pct,
         "source": "ncu --set full --clock-control none, one full-step decode_mk_kernel launch (k-permuted "
                   "planes; ncu's replay drops the cluster attribute, so the attention ran the row split -- same "
                   "bytes), 32-layer LLaMA-7B shape rho 0.6, ctx 514 (tools/gpu_final_r2b.sh, round 2 final)"}
    (OUT / "traffic.json").write_text(json.dumps(t, indent=1) + "\n")
    keys = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
            "dram__bytes_read.sum.pct_of_peak_sustained_elapsed", "dram__bytes_read.sum.per_second",
            "dram__cycles_active.sum.pct_of_peak_sustained_elapsed", "lts__t_bytes.sum",
            "sm__throughput.avg.pct_of_peak_sustained_elapsed", "launch__grid_size", "launch__cluster_dim_x",
            "launch__registers_per_thread", "sm__warps_active.avg.pct_of_peak_sustained_active"]
    with open(OUT / f"{TAG}_ncu_decode_step.txt", "w") as f:
        f.write("ncu --set full --clock-control none -k regex:decode_mk -s 2 -c 1 python tools/mk_profile_run.py 32\n")
        for k in keys:
            if k in m:
                f.write(f"{k:60s} {m[k][0]:>20s} {m[k][1]}\n")
    print("traffic.json:", t["decode_step_dram_bytes"], "bytes,", round(pct, 1), "% of DRAM peak")
