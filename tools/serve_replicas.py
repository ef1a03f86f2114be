"""C5 serving run (BASELINE.json configs[4]): N independent
requests sharded over the ranks (replicas.shard), each rank decodes its share
in waves of --wave requests through the batched engine (weights replicated, no
collective on the hot path), then the generated tokens are all-gathered to
every rank (NCCL) and rank 0 prints one JSON line.

    python tools/serve_replicas.py --requests 256 --wave 32 --prompt 1024 --gen 256
    python -m torch.distributed.run --nproc-per-node 8 --master-addr 127.0.0.1 tools/serve_replicas.py ...
"""
import argparse
import json
import sys
import time
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import paper_2605_08314_b200 as F  # noqa: E402
from paper_2605_08314_b200 import replicas  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--requests", type=int, default=256)
    ap.add_argument("--wave", type=int, default=32)
    ap.add_argument("--prompt", type=int, default=1024)
    ap.add_argument("--gen", type=int, default=256)
    ap.add_argument("--model", default="llama7b")
    ap.add_argument("--family", default="B")
    a = ap.parse_args()
    r = replicas.env_rank()
    pg = None
    torch.cuda.set_device(r.local)
    if r.world > 1:
        import torch.distributed as dist

        dist.init_process_group("nccl", device_id=torch.device("cuda", r.local))
        pg = dist
    cfg, _ = F.PRESETS[a.model]
    spec = F.SynthSpec(cfg, capacity=a.prompt + a.gen + 16, family=a.family, rho=0.6, seed=1)
    model = F.Model.synthetic(spec, dtype="bf16", device=r.local)
    mine = replicas.shard(a.requests, r.world, r.rank)
    waves = replicas.waves(mine, a.wave)
    sessions = {}
    toks = torch.zeros((len(mine), a.gen), dtype=torch.int32)
    replicas.barrier(pg)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    row = 0
    for w in waves:
        B = len(w)
        if B not in sessions:
            sessions[B] = F.Session(model, batch=B, capacity=spec.capacity, plan="full_step")
        s = sessions[B]
        s.reset()
        # request i's prompt: seeded per request (Rng64 seed 2 + i)
        prompts = np.stack([np.random.default_rng(2 + i).integers(0, cfg.vocab, a.prompt, dtype=np.int32) for i in w])
        out = s.generate(prompts, a.gen)
        toks[row: row + B] = torch.from_numpy(out)
        row += B
    torch.cuda.synchronize()
    dt = replicas.max_over_ranks(pg, time.perf_counter() - t0)
    allt = replicas.gather_rows(pg, toks, a.requests)
    if r.rank == 0:
        print(json.dumps({"workload": f"C5-style serving: {a.requests} requests x (prompt {a.prompt} + {a.gen} greedy "
                                      f"tokens), {a.model} family {a.family} rho 0.6, waves of {a.wave} per rank",
                          "n_gpus": r.world, "seconds": dt, "generated_tok_s": a.requests * a.gen / dt,
                          "tokens_gathered": list(allt.shape),
                          "token_digest": int(allt.to(torch.int64).sum().item())}))
    if pg is not None:
        pg.destroy_process_group()


if __name__ == "__main__":
    main()
