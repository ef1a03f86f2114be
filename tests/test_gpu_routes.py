"""SPEC.md ablation routes on the GPU runtime:
* lowrank_history attention: the rank-space K/V history is
  kept and the dense K, V (+ RoPE) of every cached position are rebuilt each
  decode step -- numerically the dense_kv result, reconstruction FLOPs linear
  in the cached length, dense_kv's zero.
* split plan: two graphs per layer with an explicit boundary
  copy; bitwise equal to eager, dispatches full_step < per_layer < split <
  eager, copy bytes > 0 only for split; auto FFN routing split -> no_merge."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu

TOL = {"f32": 1e-4, "bf16": 2e-2}


def _model(fsvd, dtype, seed=4):
    cfg = fsvd.ModelConfig(2, 256, 4, 64, 512, 512)
    spec = fsvd.SynthSpec(cfg, capacity=256, family="A", rho=0.5, seed=seed, conditioned=True)
    return cfg, fsvd.Model.synthetic(spec, dtype=dtype)


@pytest.mark.parametrize("dtype", ["f32", "bf16"])
def test_lowrank_history_matches_dense_kv(fsvd, oracle_mod, dtype):
    cfg, model = _model(fsvd, dtype)
    prompt = np.random.default_rng(1).integers(0, cfg.vocab, size=(1, 40), dtype=np.int32)
    outs, flops = {}, {}
    for route in ("dense_kv", "lowrank_history"):
        s = fsvd.Session(model, batch=1, capacity=256, plan="eager", attn_route=route)
        lg = [s.prefill(prompt)[0]]
        tok = int(np.argmax(lg[0]))
        fl = []
        for _ in range(12):
            before = s.stats().recon_flops
            lg.append(s.decode_step([tok])[0])
            fl.append(s.stats().recon_flops - before)
            tok = int(np.argmax(lg[-1]))
        outs[route], flops[route] = np.stack(lg), fl
    for a, b in zip(outs["lowrank_history"], outs["dense_kv"]):
        assert oracle_mod.rel_err(a, b) <= TOL[dtype]
    assert all(f == 0 for f in flops["dense_kv"])
    # per-step reconstruction FLOPs = 2 * len * (r_k + r_v) * d * L: linear in the cached length
    fl = flops["lowrank_history"]
    lens = np.arange(41, 41 + len(fl))
    assert np.array_equal(np.array(fl) * lens[0], fl[0] * lens)


def test_lowrank_history_needs_eager_plan(fsvd):
    _, model = _model(fsvd, "bf16")
    with pytest.raises(fsvd.ConfigError):
        fsvd.Session(model, batch=1, capacity=64, plan="per_layer", attn_route="lowrank_history")


def test_split_plan_counters_and_bitwise(fsvd):
    cfg, model = _model(fsvd, "f32")
    prompt = np.random.default_rng(2).integers(0, cfg.vocab, size=(1, 17), dtype=np.int32)
    res = {}
    for plan in ("eager", "split", "per_layer", "full_step"):
        s = fsvd.Session(model, batch=1, capacity=128, plan=plan, ffn="no_merge")
        lg = [s.prefill(prompt)[0]]
        st0 = s.stats()
        for _ in range(4):
            lg.append(s.decode_step([int(np.argmax(lg[-1]))])[0])
        st1 = s.stats()
        res[plan] = (np.stack(lg), (st1.dispatches - st0.dispatches) / 4, (st1.copy_bytes - st0.copy_bytes) / 4)
    for plan in ("split", "per_layer", "full_step"):
        assert np.array_equal(res[plan][0].view(np.uint32), res["eager"][0].view(np.uint32)), plan
    d = {p: r[1] for p, r in res.items()}
    assert d["full_step"] < d["per_layer"] < d["split"] < d["eager"], d
    assert d["split"] == 3 * cfg.n_layers + 1
    cb = {p: r[2] for p, r in res.items()}
    assert cb["split"] > 0
    s = fsvd.Session(model, batch=1, capacity=64, plan="split")
    assert s.resolved() == ("no_merge", "split")
