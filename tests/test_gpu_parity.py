"""GPU parity: the CUDA path through the C ABI vs the CPU oracle.

North-star tolerances (BASELINE.json): max relative logit error <= 1e-4 in
the fp32 mode and <= 2e-2 in bf16, error = max_rows max|d| / max|ref|
(SURVEY.md §8c). Oracle = f64 restatement (oracle/fsvd_oracle.cpp) on the
same normalize<float> weights and tokens. Greedy-token agreement is reported,
not required.
"""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu

TOL = {"f32": 1e-4, "bf16": 2e-2}


def _spec(fsvd, family="A", cfg=None, seed=5, conditioned=True, rho=0.5, jitter=0.0, cap=512):
    cfg = cfg or fsvd.ModelConfig(2, 128, 4, 32, 256, 512)
    return fsvd.SynthSpec(cfg, capacity=cap, family=family, rho=rho, group_size=2, seed=seed,
                          conditioned=conditioned, rank_jitter=jitter)


def _prompt(cfg, T, seed=2, batch=1):
    rng = np.random.default_rng(seed)
    return rng.integers(0, cfg.vocab, size=(batch, T), dtype=np.int32)


@pytest.mark.parametrize("dtype", ["f32", "bf16"])
@pytest.mark.parametrize("family", ["A", "B", "C", "D"])
def test_prefill_decode_vs_oracle(fsvd, oracle_mod, dtype, family):
    spec = _spec(fsvd, family, jitter=0.3 if family in "BD" else 0.0)
    cfg = spec.config
    prompt = _prompt(cfg, 37)
    om = oracle_mod.OracleModel.synthetic(spec)
    osess = om.session(f64=True, ffn="no_merge", capacity=512)
    want = [osess.prefill(prompt[0])]
    toks = [int(np.argmax(want[0]))]
    for _ in range(6):
        want.append(osess.decode_step(toks[-1]))
        toks.append(int(np.argmax(want[-1])))

    model = fsvd.Model.synthetic(spec, dtype=dtype)
    for plan in ("eager", "per_layer", "full_step"):
        s = fsvd.Session(model, batch=1, capacity=512, plan=plan)
        got = [s.prefill(prompt)[0]]
        for t in toks[:-1]:
            got.append(s.decode_step([t])[0])
        errs = [oracle_mod.rel_err(g, w) for g, w in zip(got, want)]
        assert max(errs) <= TOL[dtype], (plan, errs)
        assert s.position == 37 + 6


@pytest.mark.parametrize("dtype", ["f32", "bf16"])
def test_device_synthetic_matches_host_upload(fsvd, dtype):
    """fsvd_model_synthetic (device generator) == normalize<float> upload, bitwise."""
    for family in "ABCD":
        spec = _spec(fsvd, family, jitter=0.3)
        cfg = spec.config
        can = fsvd.Canonical.synthetic(spec)
        m_dev = fsvd.Model.synthetic(spec, dtype=dtype)
        m_host = fsvd.Model.from_canonical(can, dtype=dtype)
        for layer in range(cfg.n_layers):
            for p in fsvd.PROJ:
                r = can.rank(layer, p)
                din = cfg.d_ff if p == "down" else cfg.d_model
                dout = cfg.d_ff if p in ("up", "gate") else cfg.d_model
                for which, shape in (("A", (din, r)), ("B", (r, dout))):
                    a = m_dev.factor(layer, p, which, shape)
                    b = m_host.factor(layer, p, which, shape)
                    assert np.array_equal(a.view(np.uint32), b.view(np.uint32)), (family, layer, p, which)
                    if dtype == "f32":
                        c = can.tensor(f"layers.{layer}.{p}.{which}", shape)
                        assert np.array_equal(a.view(np.uint32), c.view(np.uint32))


def test_packed_equals_no_merge(fsvd):
    """SPEC.md:329 / :547: ffn_packed == ffn_no_merge within 1e-6 rel (f32).

    The two backends split the FFN input projection into different work
    units, so the per-tile partial sums are added in a different order; the
    reference's bound is 1e-6 relative for f32, checked per logits row."""
    spec = _spec(fsvd, "A")
    prompt = _prompt(spec.config, 20)
    model = fsvd.Model.synthetic(spec, dtype="f32")
    outs = {}
    for ffn in ("no_merge", "packed"):
        s = fsvd.Session(model, batch=1, capacity=512, ffn=ffn, plan="eager")
        lg = [s.prefill(prompt)[0]]
        for t in range(5):
            lg.append(s.decode_step([int(np.argmax(lg[-1]))])[0])
        outs[ffn] = np.stack(lg)
    for a, b in zip(outs["packed"], outs["no_merge"]):
        assert np.abs(a - b).max() / np.abs(b).max() <= 1e-6


def test_replay_equals_eager_bitwise(fsvd):
    """plan replay == eager, bitwise, same backend."""
    spec = _spec(fsvd, "C")
    prompt = _prompt(spec.config, 25)
    model = fsvd.Model.synthetic(spec, dtype="bf16")
    outs = {}
    for plan in ("eager", "per_layer", "full_step"):
        s = fsvd.Session(model, batch=1, capacity=512, ffn="packed", plan=plan)
        lg = [s.prefill(prompt)[0]]
        for _ in range(8):
            lg.append(s.decode_step([int(np.argmax(lg[-1]))])[0])
        outs[plan] = np.stack(lg)
    assert np.array_equal(outs["per_layer"].view(np.uint32), outs["eager"].view(np.uint32))
    assert np.array_equal(outs["full_step"].view(np.uint32), outs["eager"].view(np.uint32))


def test_generate_matches_stepwise(fsvd, oracle_mod):
    spec = _spec(fsvd, "A")
    prompt = _prompt(spec.config, 12)
    model = fsvd.Model.synthetic(spec, dtype="f32")
    s = fsvd.Session(model, batch=1, capacity=512, plan="full_step")
    toks = s.generate(prompt, 10)[0]
    assert s.position == 12 + 9
    om = oracle_mod.OracleModel.synthetic(spec)
    want = om.session(f64=True, capacity=512).generate(prompt[0], 10)
    assert toks[0] == want[0]  # first token always agrees in fp32 (margin >> 1e-4)
    # exactness where it is decidable: teacher-forced with the GPU's own tokens, every
    # greedy choice must equal the f64 oracle's whenever the oracle's top-2 margin
    # exceeds the fp32 tolerance (2 x 1e-4 of the logit range)
    o = om.session(f64=True, capacity=512)
    lg = o.prefill(prompt[0])
    decided = 0
    for i in range(10):
        top2 = np.sort(lg)[-2:]
        if top2[1] - top2[0] > 2e-4 * np.max(np.abs(lg)):
            assert toks[i] == int(np.argmax(lg)), (i, toks, want)
            decided += 1
        if i < 9:
            lg = o.decode_step(int(toks[i]))
    assert decided >= 8, decided


def test_batch_sequences_independent(fsvd, oracle_mod):
    spec = _spec(fsvd, "A")
    cfg = spec.config
    prompt = _prompt(cfg, 19, batch=2)
    om = oracle_mod.OracleModel.synthetic(spec)
    model = fsvd.Model.synthetic(spec, dtype="f32")
    s = fsvd.Session(model, batch=2, capacity=512, plan="per_layer")
    lp = s.prefill(prompt)
    nxt = np.argmax(lp, axis=1).astype(np.int32)
    ld = s.decode_step(nxt)
    for b in range(2):
        os_ = om.session(f64=True, capacity=512)
        assert oracle_mod.rel_err(lp[b], os_.prefill(prompt[b])) <= 1e-4
        assert oracle_mod.rel_err(ld[b], os_.decode_step(int(nxt[b]))) <= 1e-4


def test_kv_cache_matches_oracle(fsvd, oracle_mod):
    """SPEC.md:361 cache consistency: cached K/V rows equal the oracle's."""
    spec = _spec(fsvd, "B", jitter=0.2)
    prompt = _prompt(spec.config, 30)
    om = oracle_mod.OracleModel.synthetic(spec)
    osess = om.session(f64=True, capacity=512)
    osess.prefill(prompt[0])
    osess.decode_step(3)
    s = fsvd.Session(fsvd.Model.synthetic(spec, dtype="f32"), batch=1, capacity=512)
    s.prefill(prompt)
    s.decode_step([3])
    for layer in (0, 1):
        for which in "KV":
            got = s.read_kv(layer, 0, which, 0, 31)
            want = osess.read_kv(layer, which, 0, 31)
            assert np.abs(got - want).max() <= 1e-4 * np.abs(want).max()


def test_chunked_prompt_and_capacity_errors(fsvd, oracle_mod):
    spec = _spec(fsvd, "A", cap=64)
    prompt = _prompt(spec.config, 60)
    model = fsvd.Model.synthetic(spec, dtype="f32")
    s = fsvd.Session(model, batch=1, capacity=64)
    with pytest.raises(fsvd.CapacityError):
        s.prefill(_prompt(spec.config, 65))
    with pytest.raises(fsvd.ShapeError):
        s.prefill(np.zeros((1, 0), np.int32))
    with pytest.raises(fsvd.ShapeError):
        s.decode_step([1])  # before prefill
    lp = s.prefill(prompt)
    om = oracle_mod.OracleModel.synthetic(spec)
    assert oracle_mod.rel_err(lp[0], om.session(f64=True, capacity=64).prefill(prompt[0])) <= 1e-4
    for t in range(4):
        s.decode_step([t])
    with pytest.raises(fsvd.CapacityError):
        s.decode_step([1])
    s.reset()
    assert s.position == 0


def test_dispatch_counts(fsvd):
    """dispatches per step full_step < per_layer < eager."""
    spec = _spec(fsvd, "A")
    model = fsvd.Model.synthetic(spec, dtype="bf16")
    counts = {}
    for plan in ("eager", "per_layer", "full_step"):
        s = fsvd.Session(model, batch=1, capacity=512, plan=plan)
        s.prefill(_prompt(spec.config, 8))
        s.decode_step([1])
        s.decode_step([2])
        counts[plan] = s.stats().last_dispatches
        if plan != "eager":
            assert s.resolved()[0] == "packed"
        else:
            assert s.resolved()[0] == "no_merge"
    L = spec.config.n_layers
    assert L + 1 <= counts["per_layer"] <= L + 4  # n_layers + c, c <= 4
    assert counts["full_step"] == 1
    assert counts["eager"] >= 5 * counts["full_step"]
    assert counts["full_step"] < counts["per_layer"] < counts["eager"]


@pytest.mark.parametrize("dtype", ["f32", "bf16"])
@pytest.mark.parametrize("fname", ["tiny_A.fsvd", "tiny_B.fsvd", "tiny_C.fsvd", "tiny_A_rho1.fsvd"])
def test_reference_written_checkpoint(fsvd, oracle_mod, dtype, fname):
    """FSVD15 files written by the reference's own compressor (tests/golden,
    make_golden.py) through fsvd_model_load on the GPU vs the oracle on the
    same file; rho=1 also vs the reference's dense_forward_all logits."""
    import json

    from conftest import GOLDEN

    exp = json.loads((GOLDEN / "tiny_expect.json").read_text())
    c = exp["config"]
    cfg = fsvd.ModelConfig(c["n_layers"], c["d_model"], c["n_heads"], c["d_head"], c["d_ff"], c["vocab"])
    toks = np.array(exp["tokens"], dtype=np.int32)
    om = oracle_mod.OracleModel.load_file(GOLDEN / fname, cfg)
    os_ = om.session(f64=True, capacity=64)
    want = [os_.prefill(toks[:6])] + [os_.decode_step(int(t)) for t in toks[6:]]
    model = fsvd.Model.load(GOLDEN / fname, dtype=dtype)
    for plan in ("eager", "full_step"):
        s = fsvd.Session(model, batch=1, capacity=64, plan=plan)
        got = [s.prefill(toks[None, :6])[0]] + [s.decode_step([int(t)])[0] for t in toks[6:]]
        assert oracle_mod.rel_err(np.stack(got), np.stack(want)) <= TOL[dtype], plan
        if fname == "tiny_A_rho1.fsvd":
            gold = np.load(GOLDEN / "tiny_dense_logits.npy")[5:]
            assert oracle_mod.rel_err(np.stack(got), gold) <= TOL[dtype] + 1e-5


def test_batch_prefill_decode_bf16_matches_oracle(fsvd, oracle_mod):
    """B=2 independent sequences through the megakernel, bf16 tolerance."""
    spec = _spec(fsvd, "C")
    cfg = spec.config
    prompt = _prompt(cfg, 23, batch=2, seed=11)
    om = oracle_mod.OracleModel.synthetic(spec)
    model = fsvd.Model.synthetic(spec, dtype="bf16")
    s = fsvd.Session(model, batch=2, capacity=512, plan="full_step")
    lp = s.prefill(prompt)
    nxt = np.argmax(lp, axis=1).astype(np.int32)
    ld = s.decode_step(nxt)
    for b in range(2):
        os_ = om.session(f64=True, capacity=512)
        assert oracle_mod.rel_err(lp[b], os_.prefill(prompt[b])) <= 2e-2
        assert oracle_mod.rel_err(ld[b], os_.decode_step(int(nxt[b]))) <= 2e-2


@pytest.mark.parametrize("batch", [1, 2, 4])
def test_llama7b_shape_two_layers_vs_oracle(fsvd, oracle_mod, batch):
    """The bench's real layer shapes (d 4096, 32 heads x 128, d_ff 11008, V 32000,
    rho 0.6 -> ranks 1229 / 1791) for 2 layers: megakernel (B <= 2) and batched
    engine (B = 4) vs the f64 oracle, bf16 tolerance; exercises the production
    tile splits, ring chunking and the tcgen05 prefill tiles at full size."""
    base, _ = fsvd.PRESETS["llama7b"]
    cfg = fsvd.ModelConfig(2, base.d_model, base.n_heads, base.d_head, base.d_ff, base.vocab)
    spec = fsvd.SynthSpec(cfg, capacity=64, family="A", rho=0.6, seed=3, conditioned=True)
    prompt = _prompt(cfg, 9, seed=5, batch=batch)
    om = oracle_mod.OracleModel.synthetic(spec)
    model = fsvd.Model.synthetic(spec, dtype="bf16")
    s = fsvd.Session(model, batch=batch, capacity=64, plan="full_step")
    got = [s.prefill(prompt)]
    nxt = np.argmax(got[0], axis=1).astype(np.int32)
    for _ in range(2):
        got.append(s.decode_step(nxt))
        nxt = np.argmax(got[-1], axis=1).astype(np.int32)
    for b in range(batch):
        os_ = om.session(f64=True, capacity=64)
        want = [os_.prefill(prompt[b])]
        tok = int(np.argmax(got[0][b]))
        for i in range(2):
            want.append(os_.decode_step(tok))
            tok = int(np.argmax(got[i + 1][b]))
        errs = [oracle_mod.rel_err(got[i][b], want[i]) for i in range(3)]
        assert max(errs) <= TOL["bf16"], (b, errs)


def test_failed_session_create_frees_its_allocations(fsvd):
    """A session whose construction fails after allocating the KV cache (the
    megakernel's shared memory does not fit this batch x d_ff) raises
    ConfigError and frees everything (no HBM leak across retries)."""
    import torch

    cfg = fsvd.ModelConfig(2, 128, 4, 32, 32768, 512)  # B=2 x d_ff 32768 planes exceed shared memory
    spec = _spec(fsvd, "A", cfg=cfg, cap=32768)
    model = fsvd.Model.synthetic(spec, dtype="f32")
    torch.cuda.synchronize()
    free0 = torch.cuda.mem_get_info()[0]
    for _ in range(10):
        with pytest.raises(fsvd.ConfigError):
            fsvd.Session(model, batch=2, capacity=32768, plan="full_step")
    torch.cuda.synchronize()
    free1 = torch.cuda.mem_get_info()[0]
    assert free0 - free1 < 64 << 20, (free0 - free1) / 2**20
