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


def test_normalize_subcommand(tmp_path):
    """`normalize`: any family -> the normalized model as a family-A file; loading
    it back gives the same canonical tensors (family B's 1/s fold already applied)."""
    import numpy as np

    import paper_2605_08314_b200 as F
    from conftest import GOLDEN

    out = tmp_path / "a.fsvd"
    assert main(["normalize", "--ckpt", str(GOLDEN / "tiny_B.fsvd"), "--out", str(out)]) == 0
    a = F.Canonical.load_file(GOLDEN / "tiny_B.fsvd")
    b = F.Canonical.load_file(out)
    cfg = a.config
    for layer in range(cfg.n_layers):
        for p in F.PROJ:
            r = a.rank(layer, p)
            din = cfg.d_ff if p == "down" else cfg.d_model
            x = a.tensor(f"layers.{layer}.{p}.A", (din, r))
            y = b.tensor(f"layers.{layer}.{p}.A", (din, r))
            assert np.array_equal(x.view(np.uint32), y.view(np.uint32))
    assert main(["normalize", "--ckpt", str(GOLDEN / "tiny_B.fsvd")]) == 1  # --out missing: runtime error


@pytest.mark.gpu
def test_bench_csv_prompt_file_and_sweeps(tmp_path):
    import csv

    from paper_2605_08314_b200.__main__ import CSV_COLUMNS

    pf = tmp_path / "p.txt"
    pf.write_text(" ".join(str(i * 7 % 1000) for i in range(24)) + "\n")
    assert main(["generate", "--preset", "desk", "--prompt-file", str(pf), "--gen", "4", "--attn-route",
                 "lowrank_history", "--plan", "eager"]) == 0
    c = tmp_path / "r.csv"
    assert main(["bench", "--preset", "desk", "--prompt-len", "32", "--gen", "8", "--plan", "split", "--csv", str(c)]) == 0
    rows = list(csv.DictReader(open(c)))
    assert list(rows[0].keys()) == CSV_COLUMNS and rows[0]["plan"] == "split"
    assert float(rows[0]["decode_p10"]) <= float(rows[0]["decode_ms_per_token_med"]) <= float(rows[0]["decode_p90"])
    j = tmp_path / "s.json"
    assert main(["sweep-cached-len", "--preset", "desk", "--lengths", "64,128,256", "--gen", "4", "--runs", "3",
                 "--json", str(j)]) == 0
    r = json.loads(j.read_text())["rows"]
    fl = {(x["prompt_len"], x["attn_route"]): x["recon_flops_per_step"] for x in r["records"]}
    assert fl[(64, "dense_kv")] == fl[(256, "dense_kv")] == 0
    assert fl[(128, "lowrank_history")] > 1.9 * fl[(64, "lowrank_history")]  # ~linear in the cached length
    j2 = tmp_path / "ratio.json"
    assert main(["sweep-ratio", "--preset", "desk", "--rhos", "0.4,0.8", "--prompt-len", "32", "--gen", "8",
                 "--runs", "3", "--json", str(j2)]) == 0
    rr = json.loads(j2.read_text())["rows"]
    assert len(rr) == 2 and all(x["speedup"] > 0 for x in rr)
    assert rr[0]["factorized_params"] < rr[1]["factorized_params"]
