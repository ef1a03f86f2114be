#!/usr/bin/env python3
"""Benchmark: SVD-compressed LLaMA-7B-shape decoder, decode + prefill on B200.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]

Workload (BASELINE.json configs[1], "C2"): LLaMA-7B shape (L=32, d=4096,
H=32, d_ff=11008, V=32000), SVD-LLM v1 factorization (family A) at parameter
ratio 0.6 (ranks 1229 / 1791 via rank_for_ratio), random-init synthetic
weights generated on the device (seeded SplitMix64, include/fsvd/synth.hpp),
bf16 weights / fp32 accumulation, batch 1, prompt 512, decode 256.

One "step" = one request: prefill(512) + 256 greedy decode steps (argmax on
device, no host sync), all inputs resident in HBM. value = decode tokens/s
(whole job: sum over ranks); prefill tokens/s and the HBM-roofline fraction
are reported beside it. Weights (8.3 GB) exceed L2 (126 MB), so no explicit
L2 flush is needed between steps.

Multi-GPU: `--gpus N` (N > 1) re-launches itself under torch.distributed.run
(one process per GPU, NCCL, 127.0.0.1) unless already launched that way.
Requests are independent and weights are replicated, so each rank runs its own
C2 replica ("scaling": "weak"); NCCL is used only for the start barrier, the
max-over-ranks timing reduction and the result gather. The C5 leg (BASELINE.json
configs[4]) is a strong-scaling serving job: 256 requests x (prompt 1024 + 256
greedy tokens), family B, sharded over the ranks (replicas.shard) in waves of 32,
tokens all-gathered and digested (c5_tok_s, c5_frac, c5_token_digest: equal at
every N).
"""
from __future__ import annotations

import argparse
import json
import os
import subprocess
import sys
import threading
import time
from pathlib import Path

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

PROMPT, GEN, BATCH = 512, 256, 1
FAMILY, RHO, SEED = "A", 0.6, 1

# BASELINE.json configs: model preset, factorization family,
# prompt, decode horizon, batch per GPU. c2 is the headline; the others are
# measured with --config for the record (the batched engine serves B > 2).
CONFIGS = {
    "c2": dict(model="llama7b", family="A", prompt=512, gen=256, batch=1,
               desc="C2: LLaMA-7B-shape SVD-LLM v1 (family A) rho=0.6, prompt 512, decode 256, batch 1"),
    "c3": dict(model="llama7b", family="C", prompt=2048, gen=512, batch=8,
               desc="C3: LLaMA-7B-shape Basis-Sharing (family C, groups of 2) rho=0.6, prompt 2048, decode 512, batch 8"),
    "c4": dict(model="llama13b", family="D", prompt=512, gen=4096, batch=16,
               desc="C4: LLaMA-13B-shape activation-truncated (family D) rho=0.6, prompt 512, decode 4096, batch 16"),
    "c5": dict(model="llama7b", family="B", prompt=1024, gen=256, batch=32,
               desc="C5: LLaMA-7B-shape SVD-LLM v2 (family B) rho=0.6, 256 requests as waves of 32 per GPU, "
                    "prompt 1024, decode 256"),
}


def parse():
    p = argparse.ArgumentParser()
    p.add_argument("--gpus", type=int, default=1)
    p.add_argument("--steps", type=int, default=3)
    p.add_argument("--warmup", type=int, default=3)
    p.add_argument("--impl", default="ours", choices=["ours", "reference"])
    p.add_argument("--config", default="c2", choices=sorted(CONFIGS))
    p.add_argument("--prompt", type=int, default=None)
    p.add_argument("--gen", type=int, default=None)
    p.add_argument("--batch", type=int, default=None)
    p.add_argument("--plan", default="full_step", choices=["eager", "per_layer", "full_step"])
    p.add_argument("--no-cpu-baseline", action="store_true")
    p.add_argument("--cpu-steps", type=int, default=6, help="decode steps in the bounded CPU sample")
    p.add_argument("--no-c5", action="store_true", help="skip the C5 strong-scaling serving leg")
    p.add_argument("--c5-requests", type=int, default=256)
    p.add_argument("--c5-wave", type=int, default=32)
    a = p.parse_args()
    c = CONFIGS[a.config]
    a.prompt = c["prompt"] if a.prompt is None else a.prompt
    a.gen = c["gen"] if a.gen is None else a.gen
    a.batch = c["batch"] if a.batch is None else a.batch
    a.model, a.family = c["model"], c["family"]
    a.workload = c["desc"]
    if (a.prompt, a.gen, a.batch) != (c["prompt"], c["gen"], c["batch"]):
        a.workload += f" [overridden: prompt {a.prompt}, decode {a.gen}, batch {a.batch}]"
    return a


def peaks():
    try:
        j = json.loads((ROOT / "MEASURED_PEAKS.json").read_text())
        return float(j["hbm_gbs"]), float(j["bf16_tflops"]), float(j.get("bf16_tflops_sustained", j["bf16_tflops"])), "measured"
    except Exception:
        return 6650.0, 1590.0, 1400.0, "fallback"


def host_info() -> dict:
    model = "unknown"
    try:
        for line in Path("/proc/cpuinfo").read_text().splitlines():
            if line.startswith("model name"):
                model = line.split(":", 1)[1].strip()
                break
    except OSError:
        pass
    return {"cpu": model, "nproc": os.cpu_count() or 1}


def relaunch_distributed(args) -> None:
    """`--gpus N` without a torchrun environment: re-exec this script as N
    ranks (one process per GPU) under torch.distributed.run on 127.0.0.1."""
    import socket

    sk = socket.socket()
    sk.bind(("127.0.0.1", 0))
    port = sk.getsockname()[1]
    sk.close()
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
           "--master-addr", "127.0.0.1", "--master-port", str(port), str(Path(__file__).resolve()), *sys.argv[1:]]
    os.execv(sys.executable, cmd)


class Clocks:
    """nvidia-smi sampler running during the timed region."""

    def __init__(self, index: int):
        self.samples = []
        self.proc = None
        self.index = index

    def __enter__(self):
        q = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.hw_slowdown,"
             "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
             "clocks_event_reasons.sw_power_cap")
        try:
            self.proc = subprocess.Popen(["nvidia-smi", "-i", str(self.index), f"--query-gpu={q}",
                                          "--format=csv,noheader,nounits", "-lms", "200"],
                                         stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
        except Exception:
            self.proc = None
        return self

    def __exit__(self, *a):
        if self.proc is None:
            return
        self.proc.terminate()
        out, _ = self.proc.communicate(timeout=10)
        for line in out.strip().splitlines():
            f = [x.strip() for x in line.split(",")]
            if len(f) >= 7:
                try:
                    self.samples.append((float(f[0]), float(f[1]), float(f[2]), f[3:7]))
                except ValueError:
                    pass

    def summary(self):
        if not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"]}
        load = [s for s in self.samples if s[2] > 300] or self.samples
        sm = sorted(s[0] for s in load)
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for s in load for i, v in enumerate(s[3]) if v.lower().startswith("active")})
        return {"sm_mhz": sm[len(sm) // 2], "sm_max_mhz": max(s[1] for s in load), "reasons": reasons,
                "samples": len(load)}


def dist_init():
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    pg = None
    if world > 1:
        import torch
        import torch.distributed as dist

        torch.cuda.set_device(local)
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
        pg = dist
    return world, rank, local, pg


def max_over_ranks(pg, v: float) -> float:
    if pg is None:
        return v
    import torch

    t = torch.tensor([v], dtype=torch.float64, device="cuda")
    pg.all_reduce(t, op=pg.ReduceOp.MAX)
    return float(t.item())


def barrier(pg):
    if pg is not None:
        import torch

        t = torch.zeros(1, device="cuda")
        pg.all_reduce(t)
        torch.cuda.synchronize()


def spec_c2(fsvd, prompt, gen, model="llama7b", family=FAMILY):
    cfg, _ = fsvd.PRESETS[model]
    return fsvd.SynthSpec(cfg, capacity=max(1024, prompt + gen + 64), family=family, rho=RHO, seed=SEED)


# ------------------------------------------------------------- CPU baseline --
def cpu_sample(spec, steps: int, threads: int, use_ref: bool):
    """Reference CPU path on a bounded sample: prefill of a 1-token prompt,
    then `steps` decode steps, per session; `threads` independent sessions on
    `threads` cores. The runtime is the SPEC restatement in oracle/ (the
    reference has no prefill/decode code), its f32 gemv is the reference's own
    kern::Ops AVX2 kernel from oracle/_ref when available."""
    import numpy as np

    import oracle

    oracle.set_threads(16)
    om = oracle.OracleModel.synthetic(spec)
    kind = "port"
    if use_ref and oracle.ref_available():
        r = oracle.ref()
        oracle.lib().oracle_set_ref_gemv(r.ref_gemv_f32_ptr())
        kind = "reference"
    oracle.set_threads(1)
    sessions = [om.session(f64=False, ffn="no_merge", capacity=steps + 4) for _ in range(threads)]
    for s in sessions:
        s.prefill(np.array([1], np.int32))
    times = [0.0] * threads

    def run(i):
        t0 = time.perf_counter()
        tok = 1
        for _ in range(steps):
            lg = sessions[i].decode_step(tok)
            tok = int(np.argmax(lg))
        times[i] = time.perf_counter() - t0

    ths = [threading.Thread(target=run, args=(i,)) for i in range(threads)]
    for t in ths:
        t.start()
    for t in ths:
        t.join()
    wall = max(times)
    value = threads * steps / wall
    return {"value": value, "unit": "tok/s", "cores": threads, "kind": kind,
            "sample": f"{threads} independent f32 sessions x (1-token prefill + {steps} decode steps), "
                      f"LLaMA-7B-shape family A rho=0.6; gemv = {'reference kern::Ops ' + oracle.ref().ref_active_variant().decode() if kind == 'reference' else 'oracle scalar'}",
            "seconds": wall}


def run_reference(args):
    """The reference's CPU path on the box's host cores (rank 0 only): the SPEC
    runtime restated in oracle/ with the reference's own kern::Ops<float> AVX2
    gemv (oracle/_ref) -- one independent session per core, each prefilled with
    a 32-token prompt (setup, untimed), then `warmup` untimed and `steps` timed
    decode steps; one step = one greedy token on every session."""
    import numpy as np

    import oracle

    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    import paper_2605_08314_b200 as fsvd  # only for the shared config/spec dataclasses

    spec = spec_c2(fsvd, args.prompt, args.gen)
    cores = os.cpu_count() or 1
    prompt_len = 32
    oracle.set_threads(cores)
    om = oracle.OracleModel.synthetic(spec)
    sessions = [om.session(f64=False, ffn="no_merge", capacity=prompt_len + args.warmup + args.steps + 4)
                for _ in range(cores)]
    rng = np.random.default_rng(2)
    toks = []
    for s_ in sessions:  # setup: the oracle's row-batched prefill (not timed)
        toks.append(int(np.argmax(s_.prefill(rng.integers(0, spec.config.vocab, prompt_len, dtype=np.int32)))))
    kind = "port"
    if oracle.ref_available():
        oracle.lib().oracle_set_ref_gemv(oracle.ref().ref_gemv_f32_ptr())
        kind = "reference"
    oracle.set_threads(1)
    step_s = [[0.0] * cores for _ in range(args.warmup + args.steps)]

    def run(i):
        tok = toks[i]
        for k in range(args.warmup + args.steps):
            t0 = time.perf_counter()
            tok = int(np.argmax(sessions[i].decode_step(tok)))
            step_s[k][i] = time.perf_counter() - t0

    ths = [threading.Thread(target=run, args=(i,)) for i in range(cores)]
    t_all = time.perf_counter()
    for t in ths:
        t.start()
    for t in ths:
        t.join()
    t_all = time.perf_counter() - t_all
    timed = [max(step_s[k]) for k in range(args.warmup, args.warmup + args.steps)]  # slowest core per step
    wall = sum(timed)
    value = cores * args.steps / wall
    ms = sorted(1e3 * x for x in timed)
    sample = (f"{cores} independent f32 sessions (one per core) x (32-token prompt, {args.warmup} warm-up + "
              f"{args.steps} timed greedy decode steps at context {prompt_len}-{prompt_len + args.warmup + args.steps}), "
              f"LLaMA-7B-shape family A rho=0.6 (32 layers, V 32000); gemv = "
              f"{'reference kern::Ops ' + oracle.ref().ref_active_variant().decode() if kind == 'reference' else 'oracle scalar'}")
    line = {"metric": "decode tok/s, LLaMA-7B-shape SVD rank 0.6", "value": value, "unit": "tok/s",
            "impl": "reference", "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": wall * 1e3 / args.steps,
            "ms_per_step_p10_p50_p90": [ms[len(ms) // 10], ms[len(ms) // 2], ms[min(len(ms) - 1, len(ms) * 9 // 10)]],
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f32", "data": "synthetic",
            "config": {"workload": args.workload + " -- reference CPU path, bounded sample", "batch": 1},
            "host": host_info(),
            "cpu_baseline": {"value": value, "unit": "tok/s", "cores": cores, "kind": kind, "sample": sample},
            "e2e": {"value": value, "unit": "tok/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
            "run_seconds": t_all}
    print(json.dumps(line), flush=True)


# --------------------------------------------------------------- GPU bench --
def run_ours(args):
    import numpy as np
    import torch

    world, rank, local, pg = dist_init()
    torch.cuda.set_device(local)
    import paper_2605_08314_b200 as fsvd

    hbm, tf_burst, tf_sust, peak_src = peaks()
    spec = spec_c2(fsvd, args.prompt, args.gen, args.model, args.family)
    B, P, G = args.batch, args.prompt, args.gen
    model = fsvd.Model.synthetic(spec, dtype="bf16", device=local)
    info = model.info()
    cfg = info["config"]
    sess = fsvd.Session(model, batch=B, capacity=spec.capacity, plan=args.plan)
    engine = sess.engine()
    stream = torch.cuda.ExternalStream(sess.stream, device=local)
    rng = np.random.default_rng(2 + rank)
    prompts = torch.tensor(rng.integers(0, cfg.vocab, size=(B, P), dtype=np.int32), device=f"cuda:{local}")

    def one_request(ev=None):
        sess.reset()
        if ev:
            ev[0].record(stream)
        sess.prefill_device(prompts.data_ptr(), P)
        if ev:
            ev[1].record(stream)
        sess.decode_steps_device(G)  # G greedy steps on the device (megakernel: one launch per <= 256 steps)
        if ev:
            ev[2].record(stream)

    for _ in range(args.warmup):
        one_request()
    sess.sync()
    barrier(pg)
    torch.cuda.synchronize()
    evs = [[torch.cuda.Event(enable_timing=True) for _ in range(3)] for _ in range(args.steps)]
    with Clocks(local) as clk:
        t_start = torch.cuda.Event(enable_timing=True)
        t_end = torch.cuda.Event(enable_timing=True)
        t_start.record(stream)
        for k in range(args.steps):
            one_request(evs[k])
        t_end.record(stream)
        sess.sync()
        torch.cuda.synchronize()
    total_ms = t_start.elapsed_time(t_end)
    pre_ms = [e[0].elapsed_time(e[1]) for e in evs]
    dec_ms = [e[1].elapsed_time(e[2]) for e in evs]
    dec_total = max_over_ranks(pg, sum(dec_ms))
    pre_total = max_over_ranks(pg, sum(pre_ms))
    total_ms = max_over_ranks(pg, total_ms)
    barrier(pg)

    decode_tok_s = world * B * G * args.steps / (dec_total / 1e3)
    per_tok = sorted(m / G for m in dec_ms)  # per-request decode ms/token (SPEC.md:528 median, p10, p90)
    pct = [per_tok[len(per_tok) // 10], per_tok[len(per_tok) // 2], per_tok[min(len(per_tok) - 1, len(per_tok) * 9 // 10)]]
    prefill_tok_s = world * B * P * args.steps / (pre_total / 1e3)
    ms_per_token = dec_total / (G * args.steps)

    # roofline: the decode step (a chain of GEMV + attention launches) is HBM
    # bound; algorithmic bytes = factors + head + gammas + embedding row + KV
    # read (ctx_avg) + KV write.
    L, d = cfg.n_layers, cfg.d_model
    ctx_avg = P + (G + 1) / 2.0
    kv_bytes = B * (ctx_avg * L * 2 * d * 2 + L * 2 * d * 2)
    step_bytes = info["decode_weight_bytes"] + kv_bytes
    achieved_gbs = step_bytes / (ms_per_token / 1e3) / 1e9
    prefill_flops = B * (P * 2 * (info["decode_weight_bytes"] - cfg.vocab * d * 2 - d * 2 - (2 * L + 1) * d * 4) / 2
                         + 2 * L * P * P * d + 2 * d * cfg.vocab)
    prefill_tflops = prefill_flops / (pre_total / args.steps / 1e3) / 1e12

    # ---- end to end through the host-pointer C ABI (pinned host buffers) ----
    # per request: fsvd_prefill (host prompt in, host logits out) + G x
    # fsvd_decode_step (host token in, host logits out, host argmax) -- the
    # SPEC's end-to-end definition (includes prefill)
    hp = torch.empty((B, P), dtype=torch.int32, pin_memory=True)
    hp.copy_(prompts.cpu())
    tok = torch.zeros((B,), dtype=torch.int32, pin_memory=True)
    logits = torch.empty((B, cfg.vocab), dtype=torch.float32, pin_memory=True)
    import ctypes

    L_ = fsvd.lib()
    ip = ctypes.POINTER(ctypes.c_int32)
    fp = ctypes.POINTER(ctypes.c_float)
    logits_np, tok_np = logits.numpy(), tok.numpy()  # views of the pinned buffers (host argmax in numpy)
    e2e_s = []
    for rep in range(max(1, min(args.steps, 2)) + 1):
        sess.reset()
        t0 = time.perf_counter()
        fsvd._check(L_.fsvd_prefill(sess._h, ctypes.cast(hp.data_ptr(), ip), P, ctypes.cast(logits.data_ptr(), fp)))
        tok_np[:] = logits_np.argmax(axis=1)
        for _ in range(G):
            fsvd._check(L_.fsvd_decode_step(sess._h, ctypes.cast(tok.data_ptr(), ip),
                                            ctypes.cast(logits.data_ptr(), fp)))
            tok_np[:] = logits_np.argmax(axis=1)
        if rep > 0:
            e2e_s.append(time.perf_counter() - t0)
    e2e_req = max_over_ranks(pg, sum(e2e_s) / len(e2e_s))
    e2e = {"value": world * B * G / e2e_req, "unit": "tok/s",
           "h2d_bytes_per_step": B * P * 4 + B * 4 * G, "d2h_bytes_per_step": B * cfg.vocab * 4 * (G + 1),
           "ms_per_request": e2e_req * 1e3,
           "note": "per request: fsvd_prefill (pinned host prompt in, host logits out) + G x fsvd_decode_step "
                   "(pinned host token in, host logits out, host argmax); generated tokens / request wall time"}
    del sess
    del model

    # ---- C5: strong-scaling serving leg (BASELINE.json configs[4]) ----
    c5 = None
    if not args.no_c5 and args.config == "c2":
        from paper_2605_08314_b200 import replicas

        c5c = CONFIGS["c5"]
        P5, G5, W5, N5 = c5c["prompt"], c5c["gen"], args.c5_wave, args.c5_requests
        spec5 = fsvd.SynthSpec(fsvd.PRESETS[c5c["model"]][0], capacity=P5 + G5 + 16, family=c5c["family"], rho=RHO,
                               seed=SEED)
        model5 = fsvd.Model.synthetic(spec5, dtype="bf16", device=local)
        info5 = model5.info()
        sessions = {}

        def session_for(nb):
            if nb not in sessions:
                sessions[nb] = fsvd.Session(model5, batch=nb, capacity=spec5.capacity, plan="full_step")
            return sessions[nb]

        # warm-up: build the wave-size session (graph capture) and run one short wave
        mine = replicas.shard(N5, world, rank)
        for w in replicas.waves(mine, W5)[:1]:
            sw = session_for(len(w))
            sw.reset()
            sw.generate(np.stack([replicas.request_prompt(i, P5, cfg.vocab) for i in w]), 4)
        toks5, dt5, n_mine = replicas.serve(pg, N5, W5, P5, G5, cfg.vocab, session_for, sync=torch.cuda.synchronize)
        # roofline time of this rank's share: prefill FLOPs at the bf16 peak + decode bytes at HBM peak
        ideal = 0.0
        for w in replicas.waves(mine, W5):
            nb = len(w)
            pf = nb * (P5 * 2 * (info5["decode_weight_bytes"] - cfg.vocab * d * 2) / 2 + 2 * L * P5 * P5 * d)
            ideal += pf / (tf_burst * 1e12)
            for j in range(G5):
                ideal += (info5["decode_weight_bytes"] + nb * ((P5 + j + 1) * L * 2 * d * 2)) / (hbm * 1e9)
        ideal = max_over_ranks(pg, ideal)
        c5 = {"workload": c5c["desc"].replace("waves of 32", f"waves of {W5}"), "requests": N5,
              "c5_tok_s": N5 * G5 / dt5, "c5_seconds": dt5, "c5_frac": ideal / dt5,
              "c5_frac_def": "roofline time (prefill FLOPs / bf16 peak + decode bytes / HBM peak, this rank's waves) "
                             "/ measured wall time, max over ranks",
              "c5_token_digest": replicas.token_digest(toks5), "c5_tokens_gathered": list(toks5.shape),
              "timing": "host wall clock (perf_counter) around the rank's serving loop, torch.cuda.synchronize "
                        "on both sides, max over ranks"}
        del sessions
        del model5

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        try:
            cpu = cpu_sample(spec, args.cpu_steps, 1, use_ref=True)
            cpu.pop("seconds", None)
        except Exception as ex:  # baseline is reported, never required
            cpu = {"value": None, "unit": "tok/s", "cores": 1, "kind": "port", "sample": f"failed: {ex}"}

    if rank == 0:
        line = {
            "metric": "decode tok/s, LLaMA-7B-shape SVD rank 0.6",
            "value": decode_tok_s,
            "unit": "tok/s",
            "n_gpus": world,
            "steps": args.steps,
            "warmup": args.warmup,
            "ms_per_step": total_ms / args.steps,
            "higher_is_better": True,
            "scaling": "weak",
            "vs_baseline": None,
            "dtype": "bf16",
            "data": "synthetic (device-generated seeded random-init factors)",
            "config": {"workload": args.workload,
                       "model": f"{args.model}-shape", "family": args.family, "rho": RHO, "global_batch": B * world,
                       "prompt": P, "gen": G, "plan": args.plan, "parallelism": f"replicas x{world}",
                       "l2": "weights 8.3 GB > 126 MB L2: no flush needed"},
            "engine": engine,
            "decode_ms_per_token": ms_per_token,
            "decode_ms_per_token_p10_p50_p90": pct,
            "prefill_tok_s": prefill_tok_s,
            "prefill_ms": pre_total / args.steps,
            "prefill_tflops": prefill_tflops,
            "prefill_frac_bf16_peak": prefill_tflops / tf_burst,
            "roofline": {"bound": "hbm", "kernel": "decode step (GEMV chain + attention, one graph)",
                         "achieved": achieved_gbs, "peak": hbm, "unit": "GB/s", "frac": achieved_gbs / hbm,
                         "traffic": None, "algorithmic_bytes_per_step": step_bytes, "peak_source": peak_src},
            "e2e": e2e,
            "gpu_launches": None,
            "clocks": clk.summary(),
            "cpu_baseline": cpu,
            "host": host_info(),
        }
        if c5:
            line.update(c5)
        # our kernels in the timed region, per request: prefill = embed + per layer (2 RMSNorm,
        # 8 tcgen05 GEMMs, 1 flash attention, 2 split-K reductions at prompt 512) + gather + 2
        # length-register sets + the head/argmax megakernel; decode = one full-step megakernel
        # launch per <= 256 tokens (decode_steps_device; the phase program repeated inside the launch)
        if engine.get("batched"):
            # batched engine: prefill as above with the head as norm + GEMM + argmax + advance
            # (5 launches); decode per token = embed + per layer (2 RMSNorm, 8 GEMMs, <= 6
            # split-K reductions, 1 attention) + head (5), replayed as one graph
            prefill_launches = 1 + L * (2 + 8 + 1 + (2 if P <= 1024 else 0)) + 1 + 2 + 5
            line["gpu_launches"] = args.steps * (prefill_launches + G * (1 + L * 17 + 5))
        else:
            prefill_launches = 1 + L * (2 + 8 + 1 + (2 if P <= 1024 else 0)) + 1 + 2 + 1
            line["gpu_launches"] = args.steps * (prefill_launches + ((G + 255) // 256 if args.plan == "full_step"
                                                                     else G * (L + 2)))
        tf = ROOT / "profiles" / "traffic.json"
        if tf.exists():  # dram bytes of one full-step decode launch from an ncu --set full capture
            try:
                t = json.loads(tf.read_text())
                line["roofline"]["traffic"] = t.get("decode_step_dram_bytes")
                line["roofline"]["traffic_source"] = t.get("source")
            except Exception:
                pass
        print(json.dumps(line), flush=True)
    if pg is not None:
        pg.destroy_process_group()


def main():
    args = parse()
    world = os.environ.get("WORLD_SIZE")
    if world is None and args.gpus > 1:
        relaunch_distributed(args)  # does not return
    if world is not None and int(world) != args.gpus:
        raise SystemExit(f"bench.py: --gpus {args.gpus} but WORLD_SIZE={world}")
    if args.impl == "reference":
        run_reference(args)
    else:
        run_ours(args)


if __name__ == "__main__":
    main()
