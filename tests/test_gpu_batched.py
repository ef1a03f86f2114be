"""GPU parity of the batched decode engine (B > 2: configs C3-C5 of
BASELINE.json) against the CPU oracle, one independent oracle session per
sequence (sequences of a batch never interact).

Tolerances as in test_gpu_parity.py: max relative logit error <= 1e-4 in the
fp32 mode, <= 2e-2 in bf16.
"""
import os

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

TOL = {"f32": 1e-4, "bf16": 2e-2}


def _spec(fsvd, family="A", seed=7, jitter=0.0):
    cfg = fsvd.ModelConfig(2, 128, 4, 32, 256, 512)
    return fsvd.SynthSpec(cfg, capacity=256, family=family, rho=0.5, group_size=2, seed=seed, conditioned=True,
                          rank_jitter=jitter)


def _run_oracle(oracle_mod, spec, prompt, steps):
    """Per sequence: prefill logits, then greedy decode logits."""
    om = oracle_mod.OracleModel.synthetic(spec)
    logits, toks = [], []
    for b in range(prompt.shape[0]):
        os_ = om.session(f64=True, capacity=256)
        seq = [os_.prefill(prompt[b])]
        tk = [int(np.argmax(seq[0]))]
        for _ in range(steps):
            seq.append(os_.decode_step(tk[-1]))
            tk.append(int(np.argmax(seq[-1])))
        logits.append(seq)
        toks.append(tk)
    return logits, toks


@pytest.mark.parametrize("dtype", ["f32", "bf16"])
@pytest.mark.parametrize("batch,family", [(4, "A"), (5, "C"), (8, "B")])
def test_batched_prefill_decode_vs_oracle(fsvd, oracle_mod, dtype, batch, family):
    spec = _spec(fsvd, family, jitter=0.3 if family == "B" else 0.0)
    rng = np.random.default_rng(batch)
    prompt = rng.integers(0, spec.config.vocab, size=(batch, 21), dtype=np.int32)
    want, toks = _run_oracle(oracle_mod, spec, prompt, 4)
    model = fsvd.Model.synthetic(spec, dtype=dtype)
    for plan in ("eager", "full_step"):
        s = fsvd.Session(model, batch=batch, capacity=256, plan=plan)
        assert s.engine()["batched"]
        got = [s.prefill(prompt)]
        for i in range(4):  # teacher-forced with the oracle's greedy tokens
            got.append(s.decode_step(np.array([toks[b][i] for b in range(batch)], dtype=np.int32)))
        for b in range(batch):
            err = max(oracle_mod.rel_err(got[i][b], want[b][i]) for i in range(5))
            assert err <= TOL[dtype], (plan, b, err)
        assert s.position == 21 + 4


def test_batched_replay_equals_eager_bitwise(fsvd):
    """plan replay is bitwise identical to eager execution."""
    spec = _spec(fsvd, "A")
    model = fsvd.Model.synthetic(spec, dtype="bf16")
    prompt = np.random.default_rng(3).integers(0, spec.config.vocab, size=(6, 17), dtype=np.int32)
    outs = {}
    for plan in ("eager", "per_layer", "full_step"):
        s = fsvd.Session(model, batch=6, capacity=256, plan=plan)
        outs[plan] = s.generate(prompt, 8)
    assert np.array_equal(outs["eager"], outs["per_layer"])
    assert np.array_equal(outs["eager"], outs["full_step"])


def test_batched_generate_matches_oracle_greedy(fsvd, oracle_mod):
    spec = _spec(fsvd, "A")
    prompt = np.random.default_rng(9).integers(0, spec.config.vocab, size=(4, 15), dtype=np.int32)
    _, toks = _run_oracle(oracle_mod, spec, prompt, 7)
    s = fsvd.Session(fsvd.Model.synthetic(spec, dtype="f32"), batch=4, capacity=256, plan="full_step")
    got = s.generate(prompt, 8)
    want = np.array([t[:8] for t in toks])
    assert np.array_equal(got[:, 0], want[:, 0])
    assert float(np.mean(got == want)) >= 0.75, (got, want)


def test_batched_engine_matches_megakernel(fsvd, monkeypatch):
    """FSVD_BATCHED=1 routes B <= 2 through the batched engine: same logits as
    the megakernel within the bf16 tolerance (different kernels, same math)."""
    spec = _spec(fsvd, "A")
    model = fsvd.Model.synthetic(spec, dtype="bf16")
    prompt = np.random.default_rng(4).integers(0, spec.config.vocab, size=(2, 19), dtype=np.int32)
    s1 = fsvd.Session(model, batch=2, capacity=256, plan="full_step")
    assert s1.engine()["megakernel"]
    monkeypatch.setenv("FSVD_BATCHED", "1")
    s2 = fsvd.Session(model, batch=2, capacity=256, plan="full_step")
    assert s2.engine()["batched"]
    a, b = s1.prefill(prompt), s2.prefill(prompt)
    nxt = np.argmax(a, axis=1).astype(np.int32)
    a2, b2 = s1.decode_step(nxt), s2.decode_step(nxt)
    for x, y in ((a, b), (a2, b2)):
        err = np.max(np.abs(x - y)) / np.max(np.abs(x))
        assert err <= 2e-2, err


def test_batched_capacity_errors(fsvd):
    spec = _spec(fsvd, "A")
    s = fsvd.Session(fsvd.Model.synthetic(spec, dtype="bf16"), batch=4, capacity=24, plan="full_step")
    prompt = np.zeros((4, 22), dtype=np.int32)
    s.prefill(prompt)
    s.decode_step(np.zeros(4, dtype=np.int32))
    s.decode_step(np.zeros(4, dtype=np.int32))
    with pytest.raises(fsvd.CapacityError):
        s.decode_step(np.zeros(4, dtype=np.int32))


@pytest.mark.parametrize("batch", [3, 16])
def test_batched_flash_decode_dh128_vs_oracle(fsvd, oracle_mod, batch):
    """d_head 128 routes the batched decode attention through the split-KV
    flash-decode kernels (attn_decode); bf16 tolerance, teacher-forced."""
    cfg = fsvd.ModelConfig(2, 256, 2, 128, 512, 512)
    spec = fsvd.SynthSpec(cfg, capacity=256, family="A", rho=0.5, seed=13, conditioned=True)
    rng = np.random.default_rng(batch)
    prompt = rng.integers(0, cfg.vocab, size=(batch, 70), dtype=np.int32)
    want, toks = _run_oracle(oracle_mod, spec, prompt, 5)
    model = fsvd.Model.synthetic(spec, dtype="bf16")
    for plan in ("eager", "full_step"):
        s = fsvd.Session(model, batch=batch, capacity=256, plan=plan)
        got = [s.prefill(prompt)]
        for i in range(5):
            got.append(s.decode_step(np.array([toks[b][i] for b in range(batch)], dtype=np.int32)))
        for b in range(batch):
            err = max(oracle_mod.rel_err(got[i][b], want[b][i]) for i in range(6))
            assert err <= TOL["bf16"], (plan, b, err)
