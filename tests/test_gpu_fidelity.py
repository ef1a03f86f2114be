"""SPEC.md:503-511 fidelity audit on the GPU: 20 seeded prompts x 64 greedy
tokens, gold = the f64 oracle (cached; cached == no-cache is pinned in
test_oracle.py), candidates = the GPU path in f32 eager and f32 per-layer
plan (plus bf16 full-step, reported). Tolerance-free invariants of the SPEC
examples are asserted; the match rates are reported (greedy agreement is
"reported but not required", BASELINE.json north star)."""
import json

import numpy as np
import pytest

@pytest.mark.gpu
def test_fidelity_audit(fsvd, oracle_mod, tmp_path):
    from paper_2605_08314_b200 import audit

    cfg = fsvd.ModelConfig(4, 256, 8, 32, 1024, 1024)  # the reference's desk config
    spec = fsvd.SynthSpec(cfg, capacity=256, family="A", rho=0.5, seed=1, conditioned=True)
    prompts = audit.audit_prompts(20, cfg.vocab, seed=2)
    assert all(16 <= len(p) <= 128 for p in prompts)
    om = oracle_mod.OracleModel.synthetic(spec)
    gold = []
    for p in prompts:
        os_ = om.session(f64=True, capacity=256)
        gold.append(os_.generate(p, 64))
    m32 = fsvd.Model.synthetic(spec, dtype="f32")
    eager = audit.generate_candidates(m32, prompts, 64, plan="eager")
    per_layer = audit.generate_candidates(m32, prompts, 64, plan="per_layer")
    r32 = audit.score(gold, eager, per_layer)
    rbf = audit.score(gold, audit.generate_candidates(fsvd.Model.synthetic(spec, dtype="bf16"), prompts, 64,
                                                      plan="full_step"))
    print(json.dumps({"f32_eager_vs_gold": r32.as_dict(), "bf16_full_step_vs_gold": rbf.as_dict()}))
    # SPEC.md:509-510 invariants
    assert r32.first_token_match >= r32.exact_match
    assert 0.0 <= r32.mean_token_match <= 1.0
    assert r32.pairwise_exact == 20  # eager and per-layer plan are bitwise equivalent
    assert r32.first_token_match == 20  # fp32 logits within 1e-4 of the gold at the first step
    assert rbf.first_token_match >= rbf.exact_match


def test_audit_scoring_and_prompts():
    from paper_2605_08314_b200 import audit

    g = [np.array([1, 2, 3, 4]), np.array([5, 6, 7, 8])]
    c = [np.array([1, 2, 3, 4]), np.array([5, 0, 7, 0])]
    r = audit.score(g, c, c)
    assert (r.exact_match, r.first_token_match, r.pairwise_exact) == (1, 2, 2)
    assert r.mean_token_match == pytest.approx(0.75)
    a, b = audit.audit_prompts(5, 1000, seed=7), audit.audit_prompts(5, 1000, seed=7)
    assert all(np.array_equal(x, y) for x, y in zip(a, b))


def test_audit_rng_splitmix64_kat():
    """tensor.hpp Rng64 published SplitMix64 vector (test_tensor.cpp:12-15)."""
    from paper_2605_08314_b200 import audit

    assert audit.Rng64(0).next_u64() == 0xE220A8397B1DCDAF
