"""In-situ per-kernel timings of one warm C2 prefill (512 tokens, LLaMA-7B width)
from CUPTI (torch.profiler) -- no replay, no cache flush, PDL overlap intact,
unlike an ncu launch list. Prints the prefill wall time (CUDA events, no
profiler), the per-kernel-name totals and layer 1's kernel sequence.

  python tools/pf_trace.py [--prompt 512] [--label name]
Environment knobs of the runtime (FSVD_GEMM_*) apply as usual."""
import argparse
import collections
import re
import sys
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import paper_2605_08314_b200 as F  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--prompt", type=int, default=512)
ap.add_argument("--label", default="")
ap.add_argument("--reps", type=int, default=10)
a = ap.parse_args()

cfg, _ = F.PRESETS["llama7b"]
m = F.Model.synthetic(F.SynthSpec(cfg, capacity=1024, family="A", rho=0.6, seed=1), dtype="bf16")
s = F.Session(m, batch=1, capacity=1024, plan="full_step")
p = ((np.arange(a.prompt, dtype=np.int32) * 7) % cfg.vocab)[None]
for _ in range(3):
    s.reset()
    s.prefill(p)
s.sync()
ts = []
for _ in range(a.reps):
    s.reset()
    s.sync()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    s.prefill(p)  # returns host logits: synchronizes
    e1.record()
    torch.cuda.synchronize()
    ts.append(e0.elapsed_time(e1))
ts.sort()
print(f"[{a.label}] prefill {a.prompt} tokens: median {ts[len(ts) // 2]:.3f} ms  min {ts[0]:.3f} ms")

s.reset()
s.sync()
with torch.profiler.profile(activities=[torch.profiler.ProfilerActivity.CUDA]) as prof:
    s.prefill(p)
    torch.cuda.synchronize()
evs = [e for e in prof.events() if e.device_type == torch.autograd.DeviceType.CUDA]
evs.sort(key=lambda e: e.time_range.start)
def short(n):
    n = n.replace("(anonymous namespace)::", "").replace("void ", "").replace("fsvd::k::", "")
    return re.sub(r"\(.*", "", n)[:56]


ks = [(short(e.name), e.time_range.start, e.time_range.end) for e in evs]
ks = [k for k in ks if "emcpy" not in k[0] and "emset" not in k[0]]
span = (ks[-1][2] - ks[0][1]) / 1e3
busy = sum(e - b for _, b, e in ks) / 1e3
print(f"[{a.label}] traced span {span:.3f} ms, kernel-busy {busy:.3f} ms, {len(ks)} kernels")
agg = collections.OrderedDict()
for n, b, e in ks:
    x = agg.setdefault(n, [0, 0.0])
    x[0] += 1
    x[1] += (e - b) / 1e3
for n, (c, t) in sorted(agg.items(), key=lambda kv: -kv[1][1]):
    print(f"   {c:4d} {t * 1e3:9.1f} us  {n}")
# layer 1 sequence: kernels between the 2nd and 3rd rmsnorm-led blocks
per = (len(ks) - 4) // cfg.n_layers
print(f"[{a.label}] one layer (~{per} kernels): duration, end - previous end (the kernel's share of the chain)")
base = 2 + per
for i in range(base, base + per + 1):
    n, b, e = ks[i]
    print(f"   {(e - b):7.1f} us  +{(e - ks[i - 1][2]):6.1f} us  {n}")
inc = collections.OrderedDict()
for i in range(1, len(ks)):
    x = inc.setdefault(ks[i][0], [0, 0.0])
    x[0] += 1
    x[1] += ks[i][2] - ks[i - 1][2]
print(f"[{a.label}] end-to-end increments by kernel:")
for n, (c, t) in sorted(inc.items(), key=lambda kv: -kv[1][1]):
    print(f"   {c:4d} {t:9.1f} us  {n}")
