"""GPU parity in the regimes the bench and the north-star configs run.

The smaller parity tests (test_gpu_parity.py) use toy widths and short
contexts, so several production paths never run there. This file compares
those paths with the CPU oracle:

* 7B width (d 4096, 32 x 128 heads, d_ff 11008, rho 0.6, ranks 1229 / 1791),
  2 layers, reduced vocab:
  - a 512-token prefill, which uses the M = 512 tcgen05 GEMM tiles (256-row
    BMT = 2 tiles, split-K, 4-D weight tensor maps over the 11008-wide K);
  - >= 24 decode steps at context 512+, so each megakernel attention warp
    runs several 16-key batches with the running-max rescale, through both
    attention splits (one CTA pair per head; the B*H*len row split);
  - the bench's 256-step multi-step launch (decode_steps), compared token by
    token and on the last logits.
* C1 exactly (the `tiny` preset: d_head 64, 4 layers, prompt 32 + 32) in
  fp32 (1e-4) and bf16 (2e-2).
* The C4 shape (13B width, family D, B = 16) on the batched engine at context
  2048+, so the split-KV flash decode runs at realistic split counts.

Tolerances are BASELINE.json's: max relative logit error (rel_err: max over
rows of max|d| / max|ref|) <= 1e-4 in fp32 and <= 2e-2 in bf16. Decode steps
are teacher-forced with one token sequence on both sides, so a greedy
near-tie cannot make the two runs diverge; greedy agreement is reported.
"""
import os

import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu

TOL = {"f32": 1e-4, "bf16": 2e-2}


def _threads(oracle_mod):
    oracle_mod.set_threads(os.cpu_count() or 1)


@pytest.fixture(scope="module")
def wide(fsvd, oracle_mod):
    """7B-width, 2-layer model (family A, rho 0.6) and the f64 oracle after a 512-token prefill."""
    _threads(oracle_mod)
    cfg = fsvd.ModelConfig(2, 4096, 32, 128, 11008, 4096)
    spec = fsvd.SynthSpec(cfg, capacity=1024, family="A", rho=0.6, seed=11, conditioned=True)
    om = oracle_mod.OracleModel.synthetic(spec)
    assert om.rank(0, 0) == 1229 and om.rank(0, 4) == 1791  # q, up
    model = fsvd.Model.synthetic(spec, dtype="bf16")
    prompt = np.random.default_rng(7).integers(0, cfg.vocab, size=512, dtype=np.int32)
    o64 = om.session(f64=True, ffn="packed", capacity=1024)
    pre64 = o64.prefill(prompt)
    o32 = om.session(f64=False, ffn="packed", capacity=1024)
    pre32 = o32.prefill(prompt)
    return {"cfg": cfg, "spec": spec, "om": om, "model": model, "prompt": prompt, "o64": o64, "pre64": pre64,
            "o32": o32, "pre32": pre32}


@pytest.mark.parametrize("attn", ["pairs", "rows"])
def test_7b_width_prefill512_decode32(fsvd, oracle_mod, wide, attn, monkeypatch):
    """attn = pairs: one CTA pair per head merged through DSMEM (the default at
    B*H <= grid/2); rows: the B*H*len row split with per-head piece merges (the
    path larger B*H takes), forced with FSVD_MK_ATTN_PAIRS=0."""
    if attn == "rows":
        monkeypatch.setenv("FSVD_MK_ATTN_PAIRS", "0")
    s = fsvd.Session(wide["model"], batch=1, capacity=1024, plan="full_step")
    assert s.engine()["megakernel"]
    lp = s.prefill(wide["prompt"][None])[0]
    errs = [oracle_mod.rel_err(lp, wide["pre64"])]
    # cached K/V rows of the prompt (RoPE'd in the QKV GEMM epilogue) vs the oracle
    o = wide["o64"].clone()
    for layer in (0, 1):
        for which in ("K", "V"):
            got = s.read_kv(layer, 0, which, 0, 512)
            want = o.read_kv(layer, which, 0, 512)
            assert oracle_mod.rel_err(got.reshape(1, -1), want.reshape(1, -1)) <= TOL["bf16"], (layer, which)
    # 32 decode steps from context 512 (teacher-forced with the oracle's greedy tokens)
    tok = int(np.argmax(wide["pre64"]))
    agree = 0
    for _ in range(32):
        want = o.decode_step(tok)
        got = s.decode_step([tok])[0]
        errs.append(oracle_mod.rel_err(got, want))
        agree += int(np.argmax(got) == np.argmax(want))
        tok = int(np.argmax(want))
    assert max(errs) <= TOL["bf16"], errs
    assert s.position == 512 + 32
    print(f"7B width ({attn}): max rel err {max(errs):.3e}, greedy agreement {agree}/32")


def test_7b_width_decode_steps_256(fsvd, oracle_mod, wide):
    """The bench's launch: 256 greedy steps in one megakernel launch."""
    s = fsvd.Session(wide["model"], batch=1, capacity=1024, plan="full_step")
    lp = s.prefill(wide["prompt"][None])[0]
    out = torch.zeros((1, 256), dtype=torch.int32, device="cuda")
    s.decode_steps_device(256, out.data_ptr())
    s.sync()
    toks = out.cpu().numpy()[0]
    assert s.position == 512 + 256
    last = s.decode_step([int(toks[-1])])[0]
    # oracle (threaded f32), teacher-forced with the GPU's own token sequence
    o = wide["o32"].clone()
    fed = [int(np.argmax(lp))] + [int(t) for t in toks]
    agree = 0
    for i in range(256):
        lg = o.decode_step(fed[i])
        agree += int(np.argmax(lg) == toks[i])
    want_last = o.decode_step(fed[256])
    err = oracle_mod.rel_err(last, want_last)
    print(f"256-step launch: last-step rel err {err:.3e}, greedy agreement {agree}/256")
    assert err <= TOL["bf16"]
    assert agree >= 200, agree


@pytest.mark.parametrize("dtype", ["f32", "bf16"])
def test_c1_tiny_preset(fsvd, oracle_mod, dtype):
    """C1 exactly: tiny preset (4 layers, d 256, 4 heads x 64), rho 0.5, prompt 32 + 32."""
    cfg, _ = fsvd.PRESETS["tiny"]
    assert cfg.d_head == 64
    spec = fsvd.SynthSpec(cfg, capacity=128, family="A", rho=0.5, seed=1, conditioned=True)
    om = oracle_mod.OracleModel.synthetic(spec)
    assert (om.rank(0, 0), om.rank(0, 4)) == (64, 102)  # q, up
    prompt = np.random.default_rng(2).integers(0, cfg.vocab, size=32, dtype=np.int32)
    o = om.session(f64=True, ffn="packed", capacity=128)
    want = [o.prefill(prompt)]
    toks = []
    for _ in range(32):
        toks.append(int(np.argmax(want[-1])))
        want.append(o.decode_step(toks[-1]))
    model = fsvd.Model.synthetic(spec, dtype=dtype)
    for plan in ("eager", "full_step"):
        s = fsvd.Session(model, batch=1, capacity=128, plan=plan)
        got = [s.prefill(prompt[None])[0]] + [s.decode_step([t])[0] for t in toks]
        errs = [oracle_mod.rel_err(g, w) for g, w in zip(got, want)]
        assert max(errs) <= TOL[dtype], (plan, max(errs))


def test_c4_13b_shape_batched_long_context(fsvd, oracle_mod):
    """C4 shape: 13B width (d 5120, 40 x 128 heads, d_ff 13824), family D
    (activation-truncated, heterogeneous ranks), B = 16 on the batched engine,
    context 2048+ (split-KV flash decode). The 16 rows share a 2040-token
    prefix and differ in their last 8 prompt tokens; the oracle prefills the
    prefix once and forks it per row."""
    _threads(oracle_mod)
    cfg = fsvd.ModelConfig(1, 5120, 40, 128, 13824, 2048)
    spec = fsvd.SynthSpec(cfg, capacity=2304, family="D", rho=0.6, seed=13, conditioned=True, rank_jitter=0.2)
    om = oracle_mod.OracleModel.synthetic(spec)
    B, P, S = 16, 2040, 8
    rng = np.random.default_rng(3)
    prefix = rng.integers(0, cfg.vocab, size=P, dtype=np.int32)
    suffix = rng.integers(0, cfg.vocab, size=(B, S), dtype=np.int32)
    prompt = np.concatenate([np.tile(prefix, (B, 1)), suffix], axis=1)
    base = om.session(f64=False, ffn="packed", capacity=2304)
    base.prefill(prefix)
    rows = [base.clone() for _ in range(B)]
    want_pre = np.stack([rows[b].prefill(suffix[b]) for b in range(B)])

    model = fsvd.Model.synthetic(spec, dtype="bf16")
    s = fsvd.Session(model, batch=B, capacity=2304, plan="full_step")
    eng = s.engine()
    assert eng["batched"], eng  # split-KV decode: S = attn_decode_splits(16, 40, cap) (1 at this shape: 640 CTAs)
    got_pre = s.prefill(prompt)
    errs = [oracle_mod.rel_err(got_pre, want_pre)]
    toks = np.argmax(want_pre, axis=1).astype(np.int32)
    for _ in range(4):
        want = np.stack([rows[b].decode_step(int(toks[b])) for b in range(B)])
        got = s.decode_step(toks)
        errs.append(oracle_mod.rel_err(got, want))
        toks = np.argmax(want, axis=1).astype(np.int32)
    print(f"C4 shape B=16 ctx {P + S}+: max rel err {max(errs):.3e}, splits {eng['attn_splits']}")
    assert max(errs) <= TOL["bf16"], errs
