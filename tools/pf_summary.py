"""Summarize an ncu launch list of tools/prefill_once.py (second prefill only) with the gemm_tc choices log."""
import csv, sys, re, collections
def load(mode):
    rows = list(csv.reader(open(f"gpurun_out/pf_{mode}.csv")))
    hi = [i for i, r in enumerate(rows) if "Kernel Name" in r][0]
    h = rows[hi]; ki = h.index("Kernel Name"); vi = h.index("Metric Value"); mi = h.index("Metric Name")
    ks = [(r[ki], float(r[vi].replace(",", ""))) for r in rows[hi + 1:]
          if len(r) > vi and r[mi] == "gpu__time_duration.sum"]
    logs = [l for l in open(f"gpurun_out/pf_{mode}.log") if l.startswith("gemm_tc")]
    return ks, logs
for mode in sys.argv[1:]:
    ks, logs = load(mode)
    half = len(ks) // 2
    ks2 = ks[half:]
    tot = sum(t for _, t in ks2) / 1e3
    agg = collections.OrderedDict()
    for k, t in ks2:
        n = re.sub(r"\(.*", "", k)[:40]
        a = agg.setdefault(n, [0, 0.0]); a[0] += 1; a[1] += t / 1e3
    print(f"== {mode}: second prefill kernel sum {tot:.0f} us")
    for n, (c, t) in agg.items():
        print(f"   {c:4d} {t:9.1f} us  {n}")
    # per-gemm of layer 0 (second prefill): pair log lines with gemm launches
    g2 = [(k, t) for k, t in ks2 if "gemm_tc_kernel" in k]
    lg = logs[len(logs) // 2:]
    for (k, t), l in list(zip(g2, lg))[:9]:
        print(f"   {t/1e3:7.1f} us  {l.strip()}")
