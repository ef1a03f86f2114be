"""SPEC.md:512-520 cli_main: usage errors exit 2 with help text; GPU subcommands
emit the BenchResult / AuditReport JSON schema."""
import json

import pytest

from paper_2605_08314_b200.__main__ import main


def test_usage_errors_exit_2(capsys):
    assert main([]) == 2
    assert "generate" in capsys.readouterr().out
    assert main(["nonsense"]) == 2
    assert main(["bench", "--plan", "bogus"]) == 2


@pytest.mark.gpu
def test_bench_and_graph_ablation_json(tmp_path):
    out = tmp_path / "r.json"
    assert main(["bench", "--preset", "desk", "--prompt-len", "48", "--gen", "8", "--plan", "per_layer",
                 "--json", str(out)]) == 0
    r = json.loads(out.read_text())
    d = r["decode_ms_per_token"]
    assert d["p10"] <= d["median"] <= d["p90"]
    assert r["alloc_count_per_step"] == 0 and r["prefill_ms"] > 0
    out2 = tmp_path / "g.json"
    assert main(["graph-ablation", "--preset", "desk", "--prompt-len", "48", "--gen", "8", "--json", str(out2)]) == 0
    rows = {x["plan"]: x for x in json.loads(out2.read_text())["rows"]}
    # SPEC.md:488 dispatch ordering: full step < per layer < eager
    assert rows["full_step"]["dispatch_count_per_step"] < rows["per_layer"]["dispatch_count_per_step"] \
        < rows["eager"]["dispatch_count_per_step"]


@pytest.mark.gpu
def test_generate_and_audit(tmp_path, capsys, oracle_mod):
    import numpy as np

    import paper_2605_08314_b200 as F
    from paper_2605_08314_b200.audit import audit_prompts

    assert main(["generate", "--preset", "desk", "--prompt-len", "20", "--gen", "6"]) == 0
    assert len(capsys.readouterr().out.split()) == 6
    # audit without gold is an error (SPEC.md:503-511 scores against the f64 gold) ...
    assert main(["audit", "--preset", "desk", "--dtype", "f32", "--prompts", "4", "--gen", "8"]) == 1
    out = tmp_path / "a.json"
    assert main(["audit", "--preset", "desk", "--dtype", "f32", "--prompts", "4", "--gen", "8", "--pairwise-only",
                 "--json", str(out)]) == 0
    assert json.loads(out.read_text())["pairwise_exact"] == 4
    # ... with the f64 no-cache oracle gold (same prompts / weights as the CLI: seed + 1, desk preset)
    cfg, cap = F.PRESETS["desk"]
    spec = F.SynthSpec(cfg, capacity=cap, family="A", rho=0.6, seed=1)
    om = oracle_mod.OracleModel.synthetic(spec)
    prompts = audit_prompts(4, cfg.vocab, seed=2)
    gold = np.stack([om.session(f64=True, capacity=256).generate(p, 8) for p in prompts])
    np.save(tmp_path / "gold.npy", gold)
    assert main(["audit", "--preset", "desk", "--dtype", "f32", "--prompts", "4", "--gen", "8", "--gold",
                 str(tmp_path / "gold.npy"), "--json", str(out)]) == 0
    r = json.loads(out.read_text())
    assert r["pairwise_exact"] == 4 and r["first_token_match"] >= r["exact_match"] >= 3
