"""Command-line harness (SPEC.md:512-520 cli_main) for the B200 runtime.

    python -m paper_2605_08314_b200 generate  (--ckpt F | --preset P [--family A --rho 0.6]) --prompt-len T --gen N
    python -m paper_2605_08314_b200 bench     ... --prompt-len T --gen N [--batch B] [--plan eager|per_layer|full_step]
    python -m paper_2605_08314_b200 graph-ablation ... (eager vs per_layer vs full_step)
    python -m paper_2605_08314_b200 audit     ... [--gold tokens.npy]  (pairwise plans, + gold)
    python -m paper_2605_08314_b200 normalize --ckpt in.fsvd --out a.fsvd  (any family -> family A, canonical.cpp)
    python -m paper_2605_08314_b200 sweep-ratio      ... --rhos 0.2,0.4,0.6,0.8   (Fig. 4)
    python -m paper_2605_08314_b200 sweep-cached-len ... --lengths 512,1024,2048,4096 (Fig. 8)
Common axes: --plan eager|split|per_layer|full_step, --ffn auto|no_merge|packed,
--attn-route dense_kv|lowrank_history, --dtype bf16|f32; --prompt-file (whitespace
separated token ids, one line per batch row) instead of the seeded prompt;
--csv appends the SPEC.md:534 columns, --json the full records.

Machine-readable JSON to --json, human summary to stdout; exit 0 on success,
2 on usage error, 1 on runtime error. The compressor / normalize
subcommands belong to the reference's offline toolchain (out of scope here).
Weights: an FSVD15 checkpoint (--ckpt) or the seeded synthetic generator
(--preset, device-generated, SplitMix64 like the reference's fill convention).
"""
from __future__ import annotations

import argparse
import json
import statistics
import sys
import time

import numpy as np


def _model(F, a):
    if a.ckpt:
        return F.Model.load(a.ckpt, dtype=a.dtype)
    cfg, _ = F.PRESETS[a.preset]
    spec = F.SynthSpec(cfg, capacity=a.prompt_len + a.gen + 16, family=a.family, rho=a.rho, seed=a.seed)
    return F.Model.synthetic(spec, dtype=a.dtype)


def _prompt(vocab, batch, T, seed):
    from .audit import Rng64

    r = Rng64(seed)
    return np.array([[r.next_below(vocab) for _ in range(T)] for _ in range(batch)], dtype=np.int32)


CSV_COLUMNS = ["config_id", "prompt_len", "gen_len", "attn_route", "ffn", "plan", "dtype", "prefill_ms",
               "decode_ms_per_token_med", "decode_p10", "decode_p90", "e2e_s", "dispatch_per_step", "alloc_per_step",
               "copy_bytes_per_step"]


def _csv_row(r: dict) -> dict:
    """SPEC.md:534 CSV columns of one bench record (the JSON record carries the same values)."""
    d = r["decode_ms_per_token"]
    return {"config_id": r.get("config_id", ""), "prompt_len": r["prompt_len"], "gen_len": r["gen"],
            "attn_route": r["attn_route"], "ffn": r["ffn"], "plan": r["plan"], "dtype": r["dtype"],
            "prefill_ms": r["prefill_ms"], "decode_ms_per_token_med": d["median"], "decode_p10": d["p10"],
            "decode_p90": d["p90"], "e2e_s": r["end_to_end_s"], "dispatch_per_step": r["dispatch_count_per_step"],
            "alloc_per_step": r["alloc_count_per_step"], "copy_bytes_per_step": r["copy_bytes_per_step"]}


def _write_csv(path, rows):
    import csv
    import os

    new = not os.path.exists(path)
    with open(path, "a", newline="") as f:
        w = csv.DictWriter(f, fieldnames=CSV_COLUMNS)
        if new:
            w.writeheader()
        for r in rows:
            w.writerow(_csv_row(r))


def _prompt_tokens(a, vocab, batch, T):
    if getattr(a, "prompt_file", None):
        lines = [ln.split() for ln in open(a.prompt_file) if ln.strip()]
        t = np.array([[int(x) for x in ln] for ln in lines], dtype=np.int32)
        if t.shape[0] != batch:
            raise ValueError(f"--prompt-file has {t.shape[0]} rows, --batch is {batch}")
        if (t < 0).any() or (t >= vocab).any():
            raise ValueError("--prompt-file token outside the vocabulary")
        return t
    return _prompt(vocab, batch, T, a.seed + 1)


def _decode_timed(F, model, a, plan, runs, attn_route=None, ffn=None, prompt_len=None, cap=None):
    """BenchResult fields: decode ms/token (median, p10, p90), prefill ms,
    end-to-end s, dispatches / allocs / copy bytes per step."""
    attn_route = attn_route or a.attn_route
    ffn = ffn or a.ffn
    vocab = model.info()["config"].vocab
    p = _prompt_tokens(a, vocab, a.batch, prompt_len or a.prompt_len)
    P = p.shape[1]
    cap = cap or (P + a.gen + 16)
    s = F.Session(model, batch=a.batch, capacity=cap, plan=plan, ffn=ffn, attn_route=attn_route)
    dec, pre, e2e = [], [], []
    for r in range(runs + 2):  # 2 warm-up runs
        s.reset()
        t0 = time.perf_counter()
        s.prefill(p)
        s.sync()
        t1 = time.perf_counter()
        st0 = s.stats()
        for _ in range(a.gen):
            s.decode_step_device()
        s.sync()
        t2 = time.perf_counter()
        if r >= 2:
            pre.append((t1 - t0) * 1e3)
            dec.append((t2 - t1) * 1e3 / a.gen)
            e2e.append(t2 - t0)
    st = s.stats()
    q = np.percentile(dec, [10, 50, 90])
    return {"plan": plan, "attn_route": attn_route, "ffn": s.resolved()[0], "dtype": a.dtype, "batch": a.batch,
            "prompt_len": P, "gen": a.gen, "recon_flops_per_step": (st.recon_flops - st0.recon_flops) / max(1, a.gen),
            "decode_ms_per_token": {"median": float(q[1]), "p10": float(q[0]), "p90": float(q[2])},
            "prefill_ms": statistics.median(pre), "end_to_end_s": statistics.median(e2e),
            "dispatch_count_per_step": (st.dispatches - st0.dispatches) / max(1, a.gen),
            "kernel_launches_per_step": (st.kernel_launches - st0.kernel_launches) / max(1, a.gen),
            "graph_launches_per_step": (st.graph_launches - st0.graph_launches) / max(1, a.gen),
            "alloc_count_per_step": (st.allocs - st0.allocs) / max(1, a.gen),
            "copy_bytes_per_step": (st.copy_bytes - st0.copy_bytes) / max(1, a.gen),
            "engine": s.engine()}


def _sweep_ratio(F, a):
    """per retained ratio, the best path (full-step graph, packed
    FFN, dense KV) vs the eager-naive path (eager, no_merge, lowrank_history);
    speedup = naive / best decode ms/token, parameter counts per ratio."""
    rows = []
    cfg, _ = F.PRESETS[a.preset]
    for rho in [float(x) for x in a.rhos.split(",")]:
        spec = F.SynthSpec(cfg, capacity=a.prompt_len + a.gen + 16, family=a.family, rho=rho, seed=a.seed)
        model = F.Model.synthetic(spec, dtype=a.dtype)
        best = _decode_timed(F, model, a, "full_step", a.runs, attn_route="dense_kv", ffn="packed")
        naive = _decode_timed(F, model, a, "eager", a.runs, attn_route="lowrank_history", ffn="no_merge")
        can = F.Canonical.synthetic(spec)
        params = sum(can.rank(l, p) * (((cfg.d_ff if p == "down" else cfg.d_model))
                                       + (cfg.d_ff if p in ("up", "gate") else cfg.d_model))
                     for l in range(cfg.n_layers) for p in F.PROJ)
        best["config_id"] = naive["config_id"] = f"{a.preset}-{a.family}-rho{rho}"
        r = {"rho": rho, "factorized_params": int(params),
             "best_ms_per_token": best["decode_ms_per_token"]["median"],
             "naive_ms_per_token": naive["decode_ms_per_token"]["median"],
             "speedup": naive["decode_ms_per_token"]["median"] / best["decode_ms_per_token"]["median"],
             "best": best, "naive": naive}
        rows.append(r)
        print(f"rho {rho:.2f}: {params} factor params, best {r['best_ms_per_token']:.3f} ms/token, eager-naive "
              f"{r['naive_ms_per_token']:.3f} ms/token, speedup {r['speedup']:.2f}x")
        if a.csv:
            _write_csv(a.csv, [best, naive])
    return rows


def _sweep_cached_len(F, model, a):
    """per cached length L, decode latency and reconstruction FLOPs
    per step of dense_kv vs lowrank_history (both eager, same backend otherwise),
    plus the least-squares latency slopes over the lengths."""
    lens = [int(x) for x in a.lengths.split(",")]
    cap = max(lens) + a.gen + 16
    series = {"dense_kv": [], "lowrank_history": []}
    rows = []
    for L in lens:
        for route in series:
            r = _decode_timed(F, model, a, "eager", a.runs, attn_route=route, prompt_len=L, cap=cap)
            r["config_id"] = f"{a.preset}-cached{L}-{route}"
            series[route].append(r["decode_ms_per_token"]["median"])
            rows.append(r)
            print(f"L {L:5d} {route:16s} {r['decode_ms_per_token']['median']:.3f} ms/token, "
                  f"{r['recon_flops_per_step'] / 1e9:.3f} GFLOP reconstruction / step")
    slopes = {k: float(np.polyfit(lens, v, 1)[0]) for k, v in series.items()}
    print("latency slope (ms/token per cached token): " + ", ".join(f"{k} {v:.3e}" for k, v in slopes.items()))
    if a.csv:
        _write_csv(a.csv, rows)
    return {"lengths": lens, "series": series, "slopes": slopes, "records": rows}


def main(argv=None) -> int:
    ap = argparse.ArgumentParser(prog="python -m paper_2605_08314_b200", description=__doc__.split("\n\n")[0])
    sub = ap.add_subparsers(dest="cmd")
    for name in ("generate", "bench", "graph-ablation", "audit", "normalize", "sweep-ratio", "sweep-cached-len"):
        p = sub.add_parser(name)
        p.add_argument("--ckpt")
        p.add_argument("--preset", default="desk")
        p.add_argument("--family", default="A")
        p.add_argument("--rho", type=float, default=0.6)
        p.add_argument("--seed", type=int, default=1)
        p.add_argument("--dtype", default="bf16", choices=["bf16", "f32"])
        p.add_argument("--prompt-len", type=int, default=64)
        p.add_argument("--gen", type=int, default=32)
        p.add_argument("--batch", type=int, default=1)
        p.add_argument("--plan", default="full_step", choices=["eager", "split", "per_layer", "full_step"])
        p.add_argument("--ffn", default="auto", choices=["auto", "no_merge", "packed"])
        p.add_argument("--attn-route", default="dense_kv", choices=["dense_kv", "lowrank_history"])
        p.add_argument("--prompt-file", help="whitespace-separated token ids, one line per batch row")
        p.add_argument("--out", help="normalize: output FSVD15 path")
        p.add_argument("--rhos", default="0.2,0.4,0.6,0.8")
        p.add_argument("--lengths", default="512,1024,2048,4096")
        p.add_argument("--csv", help="append SPEC.md:534 CSV rows")
        p.add_argument("--runs", type=int, default=3)
        p.add_argument("--prompts", type=int, default=20)
        p.add_argument("--gold", help="audit: .npy [prompts][gen] f64 no-cache gold greedy tokens "
                                      "(tools/audit_fidelity.py writes them from the CPU oracle)")
        p.add_argument("--pairwise-only", action="store_true",
                       help="audit without gold: report only eager vs per_layer agreement")
        p.add_argument("--json")
    try:
        a = ap.parse_args(argv)
    except SystemExit as e:
        return 2 if e.code else 0
    if not a.cmd:
        ap.print_help()
        return 2
    try:
        import paper_2605_08314_b200 as F

        if a.cmd == "normalize":  # any family -> CanonicalModel<float> -> family A file (canonical.cpp)
            if not (a.ckpt and a.out):
                raise ValueError("normalize: --ckpt and --out are required")
            can = F.Canonical.load_file(a.ckpt)
            can.write_file(a.out)
            out = {"in": a.ckpt, "out": a.out, "config": vars(can.config), "shared_bases": can.shared_count()}
            print(f"normalized {a.ckpt} -> {a.out}")
            if a.json:
                with open(a.json, "w") as f:
                    json.dump(out, f, indent=1, default=str)
            return 0
        if a.cmd == "sweep-ratio":
            out = {"rows": _sweep_ratio(F, a)}
            if a.json:
                with open(a.json, "w") as f:
                    json.dump(out, f, indent=1)
            return 0
        model = _model(F, a)
        if a.cmd == "generate":
            vocab = model.info()["config"].vocab
            pr = _prompt_tokens(a, vocab, a.batch, a.prompt_len)
            s = F.Session(model, batch=a.batch, capacity=pr.shape[1] + a.gen + 16, plan=a.plan, ffn=a.ffn,
                          attn_route=a.attn_route)
            toks = s.generate(pr, a.gen)
            out = {"tokens": toks.tolist()}
            print(" ".join(map(str, toks[0].tolist())))
        elif a.cmd == "sweep-cached-len":
            out = {"rows": _sweep_cached_len(F, model, a)}
        elif a.cmd == "bench":
            if a.runs < 3:
                raise ValueError("bench: measured_runs >= 3 (SPEC.md:455)")
            out = _decode_timed(F, model, a, a.plan, a.runs)
            print(f"decode {out['decode_ms_per_token']['median']:.3f} ms/token, prefill {out['prefill_ms']:.2f} ms, "
                  f"{out['dispatch_count_per_step']:.0f} dispatches/step")
            if a.csv:
                _write_csv(a.csv, [out])
        elif a.cmd == "graph-ablation":
            rows = [_decode_timed(F, model, a, plan, a.runs) for plan in ("eager", "split", "per_layer", "full_step")]
            if a.csv:
                _write_csv(a.csv, rows)
            base = rows[0]["decode_ms_per_token"]["median"]
            for r in rows:
                r["decode_normalized_to_eager"] = r["decode_ms_per_token"]["median"] / base
                print(f"{r['plan']:10s} decode {r['decode_ms_per_token']['median']:.3f} ms/token "
                      f"({r['decode_normalized_to_eager']:.3f} x eager), {r['dispatch_count_per_step']:.0f} dispatches/step")
            out = {"rows": rows}
        else:  # audit
            from .audit import audit_prompts, generate_candidates, score

            vocab = model.info()["config"].vocab
            prompts = audit_prompts(a.prompts, vocab, seed=a.seed + 1)
            eager = generate_candidates(model, prompts, a.gen, plan="eager")
            layer = generate_candidates(model, prompts, a.gen, plan="per_layer")
            if a.gold:
                gold = list(np.load(a.gold))
                out = score(gold, eager, layer).as_dict()
                out["gold"] = a.gold
            elif a.pairwise_only:
                out = {"n_prompts": len(prompts), "max_new": a.gen,
                       "pairwise_exact": sum(int(np.array_equal(x, y)) for x, y in zip(eager, layer)),
                       "gold": None}
            else:
                raise ValueError("audit: --gold <f64 gold tokens .npy> is required (SPEC.md:503-511 scores against "
                                 "the f64 no-cache gold; tools/audit_fidelity.py produces it), or pass --pairwise-only")
            print(json.dumps(out))
        if a.json:
            with open(a.json, "w") as f:
                json.dump(out, f, indent=1)
        return 0
    except Exception as ex:  # runtime error
        print(f"error: {ex}", file=sys.stderr)
        return 1


if __name__ == "__main__":
    sys.exit(main())
