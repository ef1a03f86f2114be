"""Command-line harness (SPEC.md:512-520 cli_main) for the B200 runtime.

    python -m paper_2605_08314_b200 generate  (--ckpt F | --preset P [--family A --rho 0.6]) --prompt-len T --gen N
    python -m paper_2605_08314_b200 bench     ... --prompt-len T --gen N [--batch B] [--plan eager|per_layer|full_step]
    python -m paper_2605_08314_b200 graph-ablation ... (eager vs per_layer vs full_step)
    python -m paper_2605_08314_b200 audit     ... [--gold tokens.npy]  (pairwise plans, + gold)

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


def _decode_timed(F, model, a, plan, runs):
    """BenchResult fields: decode ms/token (median, p10, p90), prefill ms,
    end-to-end s, dispatches / allocs / copy bytes per step."""
    cap = a.prompt_len + a.gen + 16
    s = F.Session(model, batch=a.batch, capacity=cap, plan=plan)
    vocab = model.info()["config"].vocab
    p = _prompt(vocab, a.batch, a.prompt_len, a.seed + 1)
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
    return {"plan": plan, "batch": a.batch, "prompt_len": a.prompt_len, "gen": a.gen,
            "decode_ms_per_token": {"median": float(q[1]), "p10": float(q[0]), "p90": float(q[2])},
            "prefill_ms": statistics.median(pre), "end_to_end_s": statistics.median(e2e),
            "dispatch_count_per_step": (st.dispatches - st0.dispatches) / max(1, a.gen),
            "kernel_launches_per_step": (st.kernel_launches - st0.kernel_launches) / max(1, a.gen),
            "graph_launches_per_step": (st.graph_launches - st0.graph_launches) / max(1, a.gen),
            "alloc_count_per_step": (st.allocs - st0.allocs) / max(1, a.gen),
            "copy_bytes_per_step": (st.copy_bytes - st0.copy_bytes) / max(1, a.gen),
            "engine": s.engine()}


def main(argv=None) -> int:
    ap = argparse.ArgumentParser(prog="python -m paper_2605_08314_b200", description=__doc__.split("\n\n")[0])
    sub = ap.add_subparsers(dest="cmd")
    for name in ("generate", "bench", "graph-ablation", "audit"):
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
        p.add_argument("--plan", default="full_step", choices=["eager", "per_layer", "full_step"])
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

        model = _model(F, a)
        if a.cmd == "generate":
            vocab = model.info()["config"].vocab
            s = F.Session(model, batch=a.batch, capacity=a.prompt_len + a.gen + 16, plan=a.plan)
            toks = s.generate(_prompt(vocab, a.batch, a.prompt_len, a.seed + 1), a.gen)
            out = {"tokens": toks.tolist()}
            print(" ".join(map(str, toks[0].tolist())))
        elif a.cmd == "bench":
            if a.runs < 3:
                raise ValueError("bench: measured_runs >= 3 (SPEC.md:455)")
            out = _decode_timed(F, model, a, a.plan, a.runs)
            print(f"decode {out['decode_ms_per_token']['median']:.3f} ms/token, prefill {out['prefill_ms']:.2f} ms, "
                  f"{out['dispatch_count_per_step']:.0f} dispatches/step")
        elif a.cmd == "graph-ablation":
            rows = [_decode_timed(F, model, a, plan, a.runs) for plan in ("eager", "per_layer", "full_step")]
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
