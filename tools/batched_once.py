"""C3-shaped batched decode steps (B=8, 7B family C, ctx ~2048) for ncu captures of the batched engine."""
import sys
from pathlib import Path

import numpy as np

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import paper_2605_08314_b200 as F  # noqa: E402

cfg, _ = F.PRESETS["llama7b"]
spec = F.SynthSpec(cfg, capacity=2304, family="C", rho=0.6, seed=1)
m = F.Model.synthetic(spec, dtype="bf16")
s = F.Session(m, batch=8, capacity=2304, plan="eager")
p = (np.arange(8 * 2048, dtype=np.int32).reshape(8, 2048) * 7) % cfg.vocab
s.prefill(p)
for _ in range(3):
    s.decode_step_device()
s.sync()
print("done")
