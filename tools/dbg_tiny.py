import sys
from pathlib import Path
import numpy as np
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import paper_2605_08314_b200 as F
import oracle
cfg = F.ModelConfig(1, 128, 4, 32, 256, 512)
spec = F.SynthSpec(cfg, capacity=256, family="A", rho=0.5, seed=5, conditioned=True)
prompt = (np.arange(9, dtype=np.int32) * 37) % cfg.vocab
om = oracle.OracleModel.synthetic(spec)
os_ = om.session(f64=True, capacity=256)
ref = os_.prefill(prompt)
refd = os_.decode_step(3)
for dt in ("f32",):
    m = F.Model.synthetic(spec, dtype=dt)
    s = F.Session(m, batch=1, capacity=256, plan="eager")
    lp = s.prefill(prompt[None])[0]
    print("zeros", (lp == 0).sum(), "corr", np.corrcoef(lp, ref)[0, 1], "ratio", np.median(lp / ref))
    idx = np.argsort(-np.abs(ref))[:5]
    print("top ref", idx, ref[idx], lp[idx])
    print("nonzero idx", np.nonzero(lp)[0][:40])
    ld = s.decode_step([3])[0]
    print("decode zeros", (ld == 0).sum(), "corr", np.corrcoef(ld, refd)[0, 1])
