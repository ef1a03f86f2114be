"""SPEC.md:503-511 audit_fidelity on the GPU (development tool; the gold comes
from the CPU oracle = test infrastructure): 20 seeded prompts x 64 greedy
tokens on the reference's desk config, family A rho 0.5, candidates f32 eager,
f32 per-layer plan, bf16 full-step. Prints one JSON object."""
import json
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import oracle  # noqa: E402
import paper_2605_08314_b200 as F  # noqa: E402
from paper_2605_08314_b200 import audit  # noqa: E402

cfg = F.ModelConfig(4, 256, 8, 32, 1024, 1024)
res = {}
for fam in "ABC":
    spec = F.SynthSpec(cfg, capacity=256, family=fam, rho=0.5, seed=1, conditioned=True)
    prompts = audit.audit_prompts(20, cfg.vocab, seed=2)
    om = oracle.OracleModel.synthetic(spec)
    gold = [om.session(f64=True, capacity=256).generate(p, 64) for p in prompts]
    m32 = F.Model.synthetic(spec, dtype="f32")
    e = audit.generate_candidates(m32, prompts, 64, plan="eager")
    pl = audit.generate_candidates(m32, prompts, 64, plan="per_layer")
    bf = audit.generate_candidates(F.Model.synthetic(spec, dtype="bf16"), prompts, 64, plan="full_step")
    res[f"family_{fam}"] = {"f32_eager_vs_gold (pairwise: eager vs per_layer)": audit.score(gold, e, pl).as_dict(),
                            "bf16_full_step_vs_gold (pairwise: vs f32 eager)": audit.score(gold, bf, e).as_dict()}
print(json.dumps(res, indent=1))
