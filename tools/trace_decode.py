"""Per-phase timing of one megakernel decode step (FSVD_TRACE=1).

    python tools/trace_decode.py [--layers 32] [--ctx 512]

Stamps per CTA and phase (%globaltimer): [0] barrier passed, [1] input
staged, [2] chunks reduced, [3] finalized. Prints medians over CTAs for the
phases of a middle layer and the step total.
"""
import argparse
import os
import sys
from pathlib import Path

import numpy as np

os.environ["FSVD_TRACE"] = "1"
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import paper_2605_08314_b200 as F  # noqa: E402

NAMES = ["qkvA", "qkvB", "attn", "oA", "oB", "ugA", "ugB", "dA", "dB"]


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--layers", type=int, default=32)
    ap.add_argument("--ctx", type=int, default=512)
    ap.add_argument("--dtype", default="bf16")
    ap.add_argument("--batch", type=int, default=1)
    a = ap.parse_args()
    base, _ = F.PRESETS["llama7b"]
    cfg = F.ModelConfig(a.layers, base.d_model, base.n_heads, base.d_head, base.d_ff, base.vocab)
    spec = F.SynthSpec(cfg, capacity=a.ctx + 64, family="A", rho=0.6, seed=1)
    m = F.Model.synthetic(spec, dtype=a.dtype)
    s = F.Session(m, batch=a.batch, capacity=a.ctx + 64, plan="full_step")
    print("engine", s.engine())
    s.prefill(np.tile(np.arange(a.ctx, dtype=np.int32) % cfg.vocab, (a.batch, 1)))
    for _ in range(4):
        s.decode_step_device()
    s.sync()
    tr = s.trace().astype(np.int64)  # [grid, phases, 16]
    g, nph, _ = tr.shape
    names = ["embed"] + [f"L{l}.{n}" for l in range(a.layers) for n in NAMES] + ["head", "argmax"]
    if len(names) != nph:
        names = [f"p{i}" for i in range(nph)]
    t0 = tr[:, 0, 0].min()
    med = lambda x: np.median(x, axis=0) / 1e3
    stage = med(tr[:, :, 1] - tr[:, :, 0])
    wait1 = med(tr[:, :, 2] - tr[:, :, 1])      # x staged -> warp 0's first chunk ready
    dot1 = med(tr[:, :, 7] - tr[:, :, 2])       # warp 0's first chunk compute
    chunks = med(tr[:, :, 3] - tr[:, :, 1])
    fin = med(tr[:, :, 4] - tr[:, :, 3])
    pf0 = med(tr[:, :, 5] - tr[:, :, 0])        # producer first issue of the phase, rel. to barrier passed
    pf1 = med(tr[:, :, 6] - tr[:, :, 0])        # producer last issue
    start = tr[:, :, 0].min(axis=0)
    end = tr[:, :, 4].max(axis=0)
    total = end[-1] - t0
    print(f"step total {total / 1e3:.1f} us over {nph} phases, grid {g}")
    mid = a.layers // 2
    print(f"{'phase':10s} {'stage':>6s} {'wait1':>6s} {'dot1':>6s} {'chunks':>6s} {'final':>6s} {'span':>6s} {'gap':>6s} "
          f"{'pfirst':>7s} {'plast':>7s} (us, median over CTAs; producer times rel. to barrier)")
    for i, n in enumerate(names):
        if n.startswith(f"L{mid}.") or n in ("head", "argmax", "embed"):
            gap = (start[i] - end[i - 1]) / 1e3 if i else 0.0
            print(f"{n:10s} {stage[i]:6.2f} {wait1[i]:6.2f} {dot1[i]:6.2f} {chunks[i]:6.2f} {fin[i]:6.2f} "
                  f"{(end[i] - start[i]) / 1e3:6.2f} {gap:6.2f} {pf0[i]:7.2f} {pf1[i]:7.2f}")
    ct = s.chunk_trace.astype(np.int64)
    n = int((ct[:, 0] > 0).sum())
    ct = ct[:n]
    base = tr[0, 0, 0]
    # chunks of CTA 0 in a middle layer window
    lo = n * mid // a.layers
    print("CTA 0 chunks (us rel. to step start): seq issue wait_done dot_done warp | issue->ready  ready->done")
    for q in range(lo, min(n, lo + 60)):
        i_, w_, d_, wp = ct[q]
        print(f"{q:5d} {(i_ - base) / 1e3:9.2f} {(w_ - base) / 1e3:9.2f} {(d_ - base) / 1e3:9.2f} {wp:2d} | {(w_ - i_) / 1e3:7.2f} {(d_ - w_) / 1e3:7.2f}")
    f_sum = med(tr[:, :, 8] - tr[:, :, 3])
    f_fence = med(tr[:, :, 9] - tr[:, :, 8])
    f_atom = med(tr[:, :, 10] - tr[:, :, 9])
    f_load = med(tr[:, :, 11] - tr[:, :, 10])
    f_rows = med(tr[:, :, 12] - np.maximum(tr[:, :, 11], tr[:, :, 8]))
    f_tail = med(tr[:, :, 4] - tr[:, :, 12])
    dur = (tr[:, :, 4] - tr[:, :, 0]) / 1e3
    print("per-CTA phase duration (us): median p90 max | span | start skew (max-min start)")
    for i, n in enumerate(names):
        if n.startswith(f"L{mid}.") or n == "head":
            st = tr[:, i, 0]
            print(f"{n:10s} {np.median(dur[:, i]):6.2f} {np.percentile(dur[:, i], 90):6.2f} {dur[:, i].max():6.2f} | "
                  f"{(end[i] - start[i]) / 1e3:6.2f} | {(st.max() - st.min()) / 1e3:6.2f}")
    print("finalize breakdown (warp 0, first tile): recsum  fence  atomic  pieceld  rows  tail(other warps+sync)")
    for i, n in enumerate(names):
        if n.startswith(f"L{mid}.") or n == "head":
            print(f"{n:10s} {f_sum[i]:6.2f} {f_fence[i]:6.2f} {f_atom[i]:6.2f} {f_load[i]:6.2f} {f_rows[i]:6.2f} {f_tail[i]:6.2f}")
    spans = end - start
    ia = names.index(f"L{mid}.attn") if f"L{mid}.attn" in names else None
    if ia is not None:
        d = (tr[:, ia, 4] - tr[:, ia, 0]) / 1e3
        st = (tr[:, ia, 0] - tr[:, ia, 0].min()) / 1e3
        order = np.argsort(-d)
        print("attention phase, slowest CTAs: cta dur start_offset")
        print("  " + " ".join(f"{c}:{d[c]:.2f}/{st[c]:.2f}" for c in order[:30]))
        print("  fastest: " + " ".join(f"{c}:{d[c]:.2f}" for c in order[-10:]))
    cta0_timeline(s, tr, names, mid)
    print(f"sum: stage {stage.sum():.1f} us, chunks {chunks.sum():.1f} us, finalize {fin.sum():.1f} us, "
          f"phase spans {spans.sum() / 1e3:.1f} us")



def cta0_timeline(s, tr, names, mid):
    """CTA 0: per phase of the middle layer, its chunks' ready / done times
    relative to the phase start (barrier passed)."""
    ct = s.chunk_trace.astype(np.int64)
    n = int((ct[:, 0] > 0).sum())
    ct = ct[:n]
    ph_start = tr[0, :, 0]
    ph_end = tr[0, :, 4]
    for i, nm in enumerate(names):
        if not nm.startswith(f"L{mid}."):
            continue
        t0 = ph_start[i]
        sel = [q for q in range(n) if ct[q, 1] >= t0 and ct[q, 1] <= ph_end[i]]
        print(f"{nm}: staged +{(tr[0, i, 1] - t0) / 1e3:.2f}  chunks-done +{(tr[0, i, 3] - t0) / 1e3:.2f}  "
              f"end +{(ph_end[i] - t0) / 1e3:.2f} us;  chunks (ready/done): " +
              " ".join(f"{(ct[q, 1] - t0) / 1e3:.1f}/{(ct[q, 2] - t0) / 1e3:.1f}" for q in sel))


if __name__ == "__main__":
    main()
