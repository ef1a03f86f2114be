"""One C2 prefill (512 tokens) after one warm-up prefill: for ncu launch lists of the prefill kernels."""
import sys
from pathlib import Path

import numpy as np

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import paper_2605_08314_b200 as F  # noqa: E402

cfg, _ = F.PRESETS["llama7b"]
spec = F.SynthSpec(cfg, capacity=1024, family="A", rho=0.6, seed=1)
m = F.Model.synthetic(spec, dtype="bf16")
s = F.Session(m, batch=1, capacity=1024, plan="full_step")
p = (np.arange(512, dtype=np.int32) * 7) % cfg.vocab
s.prefill(p[None])
s.reset()
s.prefill(p[None])
s.sync()
print("done")
