"""In-situ (CUPTI) kernel timeline of one batched-engine decode step (C3 shape by
default: LLaMA-7B width, family C, B = 8, context 2048): per-kernel totals and the
"end minus previous end" share of each kernel in the step's dependency chain.

  python tools/batched_trace.py [--batch 8] [--ctx 2048] [--family C] [--preset llama7b]"""
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
ap.add_argument("--batch", type=int, default=8)
ap.add_argument("--ctx", type=int, default=2048)
ap.add_argument("--family", default="C")
ap.add_argument("--preset", default="llama7b")
ap.add_argument("--plan", default="full_step")
a = ap.parse_args()

cfg, _ = F.PRESETS[a.preset]
cap = a.ctx + 64
m = F.Model.synthetic(F.SynthSpec(cfg, capacity=cap, family=a.family, rho=0.6, seed=1), dtype="bf16")
s = F.Session(m, batch=a.batch, capacity=cap, plan=a.plan)
p = (np.arange(a.batch * a.ctx, dtype=np.int32).reshape(a.batch, a.ctx) * 7) % cfg.vocab
s.prefill(p)
for _ in range(3):
    s.decode_step_device()
s.sync()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(10):
    s.decode_step_device()
s.sync()
e1.record()
torch.cuda.synchronize()
print(f"engine {s.engine()}; step {e0.elapsed_time(e1) / 10:.3f} ms (B={a.batch}, ctx {a.ctx})")

with torch.profiler.profile(activities=[torch.profiler.ProfilerActivity.CUDA]) as prof:
    s.decode_step_device()
    s.sync()
    torch.cuda.synchronize()
evs = [e for e in prof.events() if e.device_type == torch.autograd.DeviceType.CUDA]
evs.sort(key=lambda e: e.time_range.start)


def short(n):
    n = n.replace("(anonymous namespace)::", "").replace("void ", "").replace("fsvd::k::", "")
    return re.sub(r"\(.*", "", n)[:56]


ks = [(short(e.name), e.time_range.start, e.time_range.end) for e in evs]
ks = [k for k in ks if "emcpy" not in k[0] and "emset" not in k[0]]
print(f"traced span {(ks[-1][2] - ks[0][1]) / 1e3:.3f} ms, {len(ks)} kernels")
inc = collections.OrderedDict()
for i in range(len(ks)):
    x = inc.setdefault(ks[i][0], [0, 0.0, 0.0])
    x[0] += 1
    x[1] += ks[i][2] - ks[i][1]
    x[2] += ks[i][2] - (ks[i - 1][2] if i else ks[i][1])
print("   count  busy(us)  share(us)  kernel")
for n, (c, t, sh) in sorted(inc.items(), key=lambda kv: -kv[1][2]):
    print(f"   {c:5d} {t:9.1f} {sh:10.1f}  {n}")
per = len(ks) // cfg.n_layers
print("layer 1 sequence: duration, share")
for i in range(2 + per, 2 + 2 * per):
    n, b, e = ks[i]
    print(f"   {e - b:7.1f} +{e - ks[i - 1][2]:6.1f}  {n}")
