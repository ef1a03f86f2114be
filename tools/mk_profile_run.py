"""Small driver for ncu: L-layer 7B-width model, a few full-step decodes."""
import sys
from pathlib import Path
import numpy as np
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import paper_2605_08314_b200 as F
L = int(sys.argv[1]) if len(sys.argv) > 1 else 4
b, _ = F.PRESETS["llama7b"]
cfg = F.ModelConfig(L, b.d_model, b.n_heads, b.d_head, b.d_ff, b.vocab)
spec = F.SynthSpec(cfg, capacity=640, family="A", rho=0.6, seed=1)
m = F.Model.synthetic(spec, dtype="bf16")
s = F.Session(m, batch=1, capacity=640, plan="full_step")
s.prefill(np.arange(512, dtype=np.int32)[None] % cfg.vocab)
for _ in range(3):
    s.decode_step_device()
s.sync()
