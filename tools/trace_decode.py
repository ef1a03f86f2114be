"""Per-phase timing of one megakernel decode step (FSVD_TRACE=1).

    python tools/trace_decode.py [--layers 32] [--ctx 512]

Prints, per phase type of a middle layer and summed over the step: barrier
wait, input staging, tile work (median over CTAs) and the wall span of the
phase, plus bytes and achieved GB/s per phase.
"""
import argparse
import os
import sys
from pathlib import Path

import numpy as np

os.environ["FSVD_TRACE"] = "1"
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import paper_2605_08314_b200 as F  # noqa: E402

NAMES_PACKED = ["qkvA", "qkvB", "attn", "oA", "oB", "ugA", "ugB", "dA", "dB"]


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--layers", type=int, default=32)
    ap.add_argument("--ctx", type=int, default=512)
    ap.add_argument("--dtype", default="bf16")
    a = ap.parse_args()
    base, _ = F.PRESETS["llama7b"]
    cfg = F.ModelConfig(a.layers, base.d_model, base.n_heads, base.d_head, base.d_ff, base.vocab)
    spec = F.SynthSpec(cfg, capacity=a.ctx + 64, family="A", rho=0.6, seed=1)
    m = F.Model.synthetic(spec, dtype=a.dtype)
    s = F.Session(m, batch=1, capacity=a.ctx + 64, plan="full_step")
    print("engine", s.engine())
    s.prefill(np.arange(a.ctx, dtype=np.int32)[None] % cfg.vocab)
    for _ in range(4):
        s.decode_step_device()
    s.sync()
    tr = s.trace().astype(np.int64)  # [grid, phases, 8]
    g, nph, _ = tr.shape
    t0 = tr[:, 0, 0].min()
    tr = tr - t0
    names = [f"L{l}.{n}" for l in range(a.layers) for n in NAMES_PACKED] + ["head", "argmax"]
    if len(names) != nph:
        names = [f"p{i}" for i in range(nph)]
    wait = np.median(tr[:, :, 1] - tr[:, :, 0], axis=0)
    stage = np.median(tr[:, :, 2] - tr[:, :, 1], axis=0)
    work = np.median(tr[:, :, 3] - tr[:, :, 2], axis=0)
    wmax = (tr[:, :, 3] - tr[:, :, 2]).max(axis=0)
    start = tr[:, :, 1].min(axis=0)
    end = tr[:, :, 3].max(axis=0)
    total = end[-1] - tr[:, 0, 0].min()
    print(f"step total {total / 1e3:.1f} us over {nph} phases, grid {g}")
    mid = a.layers // 2
    units0 = np.median(tr[:, :, 4] - tr[:, :, 2], axis=0)
    units1 = np.median(tr[:, :, 5] - tr[:, :, 2], axis=0)
    sync = np.median(tr[:, :, 6] - np.maximum(tr[:, :, 4], tr[:, :, 5]), axis=0)
    comb = np.median(tr[:, :, 7] - tr[:, :, 6], axis=0)
    print(f"{'phase':10s} {'wait':>7s} {'stage':>7s} {'work':>7s} {'workmax':>7s} {'span':>7s} {'units0':>7s} "
          f"{'units1':>7s} {'sync':>7s} {'comb':>7s} (us, median over CTAs)")
    for i, n in enumerate(names):
        if n.startswith(f"L{mid}.") or n in ("head", "argmax"):
            print(f"{n:10s} {wait[i] / 1e3:7.2f} {stage[i] / 1e3:7.2f} {work[i] / 1e3:7.2f} {wmax[i] / 1e3:7.2f} "
                  f"{(end[i] - start[i]) / 1e3:7.2f} {units0[i] / 1e3:7.2f} {units1[i] / 1e3:7.2f} "
                  f"{sync[i] / 1e3:7.2f} {comb[i] / 1e3:7.2f}")
    print(f"sum median: wait {wait.sum() / 1e3:.1f} us, stage {stage.sum() / 1e3:.1f} us, work {work.sum() / 1e3:.1f} us")


if __name__ == "__main__":
    main()
