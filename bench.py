#!/usr/bin/env python
"""ChunkFlow B200 benchmark (BASELINE.json metric: tokens/sec on a long-tail
SFT batch at chunk 8K; peak HBM GB).

Workload (config C2): Llama-7B-shaped layer stack (d 4096, 32
layers, 32 heads, GQA-8, SwiGLU ffn 11008, vocab 32000, RMSNorm, RoPE),
random SplitMix64 init in bf16 (fp32 gradients), one step = the full chunked
forward+backward of one 1,000-sequence long-tail block per GPU: 999 sequences
log-uniform in [16,1024) + one 37,888-token sequence = 265,592 tokens, chunk
size 8192, K=1 (33 chunks, 70 events, 4 recomputed forwards), loss and fp32
parameter gradients (NCCL all-reduce across ranks for N>1).

  python bench.py [--gpus N --steps K --warmup W] [--impl reference]

One JSON line on rank 0.  `value` is device-timed (CUDA events on the
library's stream, max over ranks) with the step's inputs resident in HBM;
`e2e` goes through the public C-ABI call (cf_plan_build + cf_run_plan) with
host token buffers, host->device copies and the loss read-back inside the
timed region.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

MODEL = dict(vocab=32000, d=4096, heads=32, kv_heads=8, layers=32, ffn=11008, seed=1, rope_theta=10000.0,
             rms_eps=1e-5)
CHUNK, K_RETAIN = 8192, 1
METRIC = "tokens/sec on long-tail SFT batch (chunk 8K) at 1/2/4/8 B200; peak HBM GB"


WORKLOAD = "c2"  # c2 (the metric's workload) | long | short (profiling slices of it)


def block_lengths(seed):
    import paper_2503_02356_b200 as cf
    short = cf.capi.synthesize(999, seed, preset=0, bounds=[1024], fracs=[1.0], max_length=1024)
    if WORKLOAD == "long":
        return np.array([37888], np.int64)
    if WORKLOAD == "short":
        return short.astype(np.int64)
    return np.concatenate([short, [37888]]).astype(np.int64)


def dist_env():
    return int(os.environ.get("RANK", 0)), int(os.environ.get("WORLD_SIZE", 1)), int(os.environ.get("LOCAL_RANK", 0))


class ClockSampler:
    """nvidia-smi clocks + throttle reasons sampled during the timed region."""

    def __init__(self, gpu):
        self.gpu = gpu
        self.rows = []
        self.proc = None

    def __enter__(self):
        q = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.hw_slowdown,"
             "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
             "clocks_event_reasons.sw_power_cap")
        try:
            self.proc = subprocess.Popen(["nvidia-smi", "-i", str(self.gpu), f"--query-gpu={q}",
                                          "--format=csv,noheader,nounits", "-lms", "200"],
                                         stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except FileNotFoundError:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            parts = [p.strip() for p in line.split(",")]
            if len(parts) == 7:
                self.rows.append(parts)

    def __exit__(self, *a):
        if self.proc:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except subprocess.TimeoutExpired:
                self.proc.kill()

    def summary(self):
        if not self.rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"]}
        sm = [float(r[0]) for r in self.rows if r[0].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for r in self.rows for i in range(4) if r[3 + i] == "Active"})
        return {"sm_mhz": statistics.median(sm) if sm else None,
                "sm_max_mhz": float(self.rows[0][1]) if self.rows[0][1].replace(".", "").isdigit() else None,
                "reasons": reasons, "samples": len(self.rows)}


def peaks():
    try:
        return json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))
    except Exception:
        return {"hbm_gbs": 6650.0, "bf16_tflops": 1590.0, "bf16_tflops_sustained": 1400.0, "fallback": True}


TRAFFIC_FILE = "profiles/round2_gemm_traffic.json"


HBM_FILE = "profiles/round2_hbm_kernels.json"


def hbm_kernels():
    """Achieved GB/s of the non-contraction kernels at C2 widths from the
    committed ncu capture (tools/hbm_kernels.py): algorithmic bytes per launch
    / ncu duration, DRAM bytes, fraction of the measured copy bandwidth."""
    try:
        t = json.load(open(os.path.join(ROOT, HBM_FILE)))
    except Exception:
        return None
    ks = {k: {f: round(v[f], 3) if isinstance(v[f], float) else v[f]
              for f in ("median_us", "achieved_gbs", "dram_gbs", "frac_of_peak", "traffic_over_algorithmic")
              if f in v and v[f] is not None}
          for k, v in t["kernels"].items()}
    return {"source": HBM_FILE, "peak_gbs": t["peak_gbs"], "peak_kind": t["peak_kind"], "workload": t["workload"],
            "kernels": ks}


def gemm_traffic():
    """Per-launch DRAM bytes of the GEMM from the committed ncu --set full
    capture (tools/gemm_traffic.py), with the algorithmic bytes of the same
    launches for comparison; None when the capture is absent."""
    try:
        t = json.load(open(os.path.join(ROOT, TRAFFIC_FILE)))
        if "mean_dram_bytes_per_launch" not in t:  # tools/gemm_traffic_quick.py: one entry per variant
            t = next(v for v in t.values() if isinstance(v, dict) and "mean_dram_bytes_per_launch" in v)
        return t["mean_dram_bytes_per_launch"], t["mean_algorithmic_bytes_per_launch"]
    except Exception:
        return None, None


# ----------------------------------------------------------- CPU baseline
def toy_flops(lengths, cfg, cs):
    """Algorithmic FLOPs of the reference toy run_plan (6NT + 12*L*d*pairs)."""
    d, L, V, kvw = cfg.d_model, cfg.num_layers, cfg.vocab_size, cfg.d_model // cfg.num_heads * cfg.num_kv_heads
    N = L * (2 * d * d + 2 * d * kvw + 4 * d * d) + d * V
    pairs = 0.0
    for n in lengths:
        pairs += n * (n + 1) / 2
    return 6.0 * N * float(sum(lengths)) + 12.0 * L * d * pairs


def _c1_workload():
    from oracle.oracle import Oracle, c1_batch, c1_cfg
    o = Oracle()
    lengths, tokens = c1_batch(o)
    return lengths, tokens, c1_cfg()


def _disjoint_slices(lengths, parts):
    """LPT split of the batch's sequences into `parts` disjoint subsets by
    attention-weighted work (whole sequences, so a dependent group stays in
    one process, as on the GPU)."""
    order = np.argsort(-lengths, kind="stable")
    load = np.zeros(parts)
    out = [[] for _ in range(parts)]
    for i in order:
        w = float(lengths[i]) * (1.0 + lengths[i] / 2048.0)
        r = int(np.argmin(load))
        load[r] += w
        out[r].append(int(i))
    return [sorted(x) for x in out if x]


def cpu_reference_sample(procs=1):
    """Times the UNMODIFIED reference run_plan (oracle/_ref/libcfref.so,
    compiled from /root/reference in the build container; the oracle port
    when it is absent) on the C1 workload — toy model V256/d256/H4/KVH2/L2,
    the canonical 33-sequence C1 batch incl. its 2,048-token sequence (a
    4-chunk dependent group: prefix K/V reads, dK/dV scatter, recompute),
    chunk 512, K = 2.
      procs == 1: a bounded sample — the 2,048-token group plus the leading
                  short sequences up to ~4,000 tokens — on one core;
      procs  > 1: the FULL C1 batch split into `procs` disjoint subsets of
                  whole sequences, one process each, wall-clock over all.
    Returns C1 tokens/s and the same throughput converted to C2 tokens/s by
    algorithmic FLOPs/token (the reference cannot run a Llama-shaped model)."""
    from oracle.oracle import Oracle, Reference
    try:
        Reference()
        kind = "reference"
    except FileNotFoundError:
        kind = "port"
    lengths, tokens, cfg = _c1_workload()
    offs = np.concatenate([[0], np.cumsum(lengths)])
    if procs == 1:
        pick, tot = [len(lengths) - 1], int(lengths[-1])
        for i in range(len(lengths) - 1):
            if tot + lengths[i] > 4000:
                break
            pick.append(i)
            tot += int(lengths[i])
        slices = [sorted(pick)]
    else:
        slices = _disjoint_slices(lengths, procs)
    jobs = [(kind, lengths[s].tolist(), np.concatenate([tokens[offs[i]:offs[i + 1]] for i in s]).tolist(),
             [int(i) for i in s]) for s in slices]
    flops = sum(toy_flops(lengths[s], cfg, 512) for s in slices)
    ntok = int(sum(lengths[s].sum() for s in slices))
    if len(jobs) == 1:
        t0 = time.perf_counter()
        _ref_worker(*jobs[0])
        dt = time.perf_counter() - t0
    else:
        import multiprocessing as mp
        with mp.get_context("fork").Pool(len(jobs)) as pool:
            t0 = time.perf_counter()
            pool.starmap(_ref_worker, jobs)
            dt = time.perf_counter() - t0
    fps = flops / dt
    c2_flops_per_token = c2_flops_per_token_est()
    what = (f"bounded C1 sample: the 2,048-token group + {len(slices[0]) - 1} short sequences ({ntok} tokens), 1 core"
            if procs == 1 else f"full C1 batch ({ntok} tokens, 33 sequences) in {len(jobs)} disjoint processes")
    return {"kind": kind, "cpu_flops_per_s": fps, "seconds": dt, "sample_tokens": ntok,
            "c1_tokens_per_s": ntok / dt,
            "sample": f"reference run_plan, toy C1 model (V256 d256 H4 KVH2 L2), chunk 512, K=2 — {what}; "
                      f"tokens/s converted to C2 by algorithmic FLOPs ({c2_flops_per_token / 1e9:.1f} GFLOP/token)",
            "tokens_per_s": fps / c2_flops_per_token, "cores": len(jobs)}


def _ref_worker(kind, sl, st, ids):
    from oracle.oracle import Oracle, Reference, c1_cfg
    lib = Reference() if kind == "reference" else Oracle()
    lib.run_plan(c1_cfg(), np.array(sl), np.array(st, np.int32), 512, 2, ids=np.array(ids, np.int64))


def gpu_c1_side_by_side(ctx, steps=10):
    """The GPU on the same C1 workload (toy model, C1 batch, chunk 512, K=2)
    through the public call (plan build + cf_run_plan with host buffers),
    device-timed: the like-for-like counterpart of the CPU baseline."""
    import torch
    import paper_2503_02356_b200 as cf
    lengths, tokens, _ = _c1_workload()
    model = cf.Model(ctx, cf.model_cfg(arch=0, vocab=256, d=256, heads=4, kv_heads=2, layers=2, seed=1))
    stream = torch.cuda.ExternalStream(ctx.stream)
    for _ in range(3):
        model.run_plan(cf.Plan.build(lengths, 512, 2), lengths, tokens)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    ctx.synchronize()
    e0.record(stream)
    for _ in range(steps):
        r = model.run_plan(cf.Plan.build(lengths, 512, 2), lengths, tokens)
    e1.record(stream)
    e1.synchronize()
    model.close()
    return {"tokens_per_s": float(lengths.sum()) * steps / (e0.elapsed_time(e1) / 1e3), "loss": r.loss,
            "tokens": int(lengths.sum())}


def c2_flops_per_token_est():
    """Algorithmic FLOPs/token of the C2 block: 6N + 12*L*H*dh*pairs/tokens
    (pairs = sum len(len+1)/2 — chunking with KV state preserves the pairs)."""
    from oracle.oracle import Oracle
    d, L, H, dh, kvw, ffn, V = 4096, 32, 32, 128, 1024, 11008, 32000
    N = L * (d * (d + 2 * kvw) + d * d + d * 2 * ffn + ffn * d) + d * V
    lens = np.concatenate([Oracle().synthesize(999, 1, preset=0, bounds=[1024], fracs=[1.0], max_length=1024),
                           [37888]]).astype(np.float64)
    pairs = float((lens * (lens + 1) / 2).sum())
    return 6.0 * N + 12.0 * L * H * dh * pairs / float(lens.sum())


def run_reference_arm(args):
    rank, world, _ = dist_env()
    if rank != 0:
        return
    procs = os.cpu_count() or 1
    vals = []
    for _ in range(args.warmup):
        cpu_reference_sample(procs=procs)
    for _ in range(args.steps):
        vals.append(cpu_reference_sample(procs=procs))
    tps = statistics.median(v["tokens_per_s"] for v in vals)
    line = {"impl": "reference", "metric": METRIC, "value": tps, "unit": "tokens/s", "n_gpus": args.gpus,
            "steps": args.steps, "warmup": args.warmup, "higher_is_better": True, "scaling": "weak",
            "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": {"workload": "C2 Llama-7B-shaped long-tail block, chunk 8192, K=1 (CPU: reference toy "
                                   "run_plan, FLOP-extrapolated)", "global_batch": 1000 * args.gpus},
            "cpu_baseline": {"value": tps, "unit": "tokens/s", "cores": procs, "kind": vals[0]["kind"],
                             "sample": vals[0]["sample"]},
            "e2e": {"value": tps, "unit": "tokens/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


# ------------------------------------------------------------ B200 arm
def run_b200(args):
    import torch
    import paper_2503_02356_b200 as cf

    rank, world, local = dist_env()
    if world != args.gpus:
        raise SystemExit(f"launched with WORLD_SIZE={world} but --gpus {args.gpus}")
    torch.cuda.set_device(local)
    dist = None
    if world > 1:
        import torch.distributed as dist
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    ctx = cf.Context(local)
    if world > 1:
        uid = [cf.Context.nccl_unique_id() if rank == 0 else None]
        dist.broadcast_object_list(uid, src=0)
        ctx.init_dp(rank, world, uid[0])
    cfg = cf.model_cfg(arch=cf.ARCH_LLAMA, **{k: v for k, v in MODEL.items()})
    model = cf.Model(ctx, cfg)

    # global batch: one 1,000-sequence block per rank (weak scaling)
    blocks = [block_lengths(b + 1) for b in range(world)]
    lengths = np.concatenate(blocks)
    ids = np.arange(len(lengths), dtype=np.int64)
    tokens = np.concatenate([cf.gen_tokens(bl, MODEL["vocab"], b + 1) for b, bl in enumerate(blocks)])
    gplan = cf.Plan.build(lengths, CHUNK, K_RETAIN, ids)
    plan = gplan.partition(world, rank) if world > 1 else gplan
    step = cf.Step(model, plan, lengths, tokens, ids)
    stream = torch.cuda.ExternalStream(ctx.stream)

    def barrier():
        ctx.synchronize()
        torch.cuda.synchronize()
        if dist:
            dist.barrier()

    for _ in range(args.warmup):
        r = step.run()
    barrier()
    ctx.set_profiling(True)
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    res = []
    with ClockSampler(local) as clk:
        barrier()
        ev0.record(stream)
        for _ in range(args.steps):
            res.append(step.run())
        ev1.record(stream)
        ev1.synchronize()
        barrier()
    ctx.set_profiling(False)
    ms = ev0.elapsed_time(ev1)
    my_tokens = sum(r.tokens for r in res) / args.steps
    # e2e through the public call: plan build + H2D of the batch + loss D2H
    pinned_tok = torch.from_numpy(tokens).pin_memory().numpy()
    barrier()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    for _ in range(max(1, args.steps)):
        gp = cf.Plan.build(lengths, CHUNK, K_RETAIN, ids)
        p = gp.partition(world, rank) if world > 1 else gp
        re = model.run_plan(p, lengths, pinned_tok, ids)
    e1.record(stream)
    e1.synchronize()
    barrier()
    e2e_ms = e0.elapsed_time(e1)
    h2d = int(step.input_bytes())  # the same per-step upload cf_run_plan performs (same plan and batch)
    d2h = 8 * (p.counts()[2] + 1)

    stats = torch.tensor([ms, e2e_ms, my_tokens], dtype=torch.float64, device="cuda")
    if dist:
        t = stats.clone()
        dist.all_reduce(t[:2], op=dist.ReduceOp.MAX)
        tok = stats[2:].clone()
        dist.all_reduce(tok, op=dist.ReduceOp.SUM)
        stats = torch.cat([t[:2], tok])
    ms_max, e2e_max, tokens_all = stats.tolist()
    if rank != 0:
        if dist:
            dist.destroy_process_group()
        return
    pk = peaks()
    traffic = gemm_traffic()
    r0 = res[-1]
    gemm_tf = sum(r.gemm_flops for r in res) / (sum(r.gemm_ms for r in res) / 1e3) / 1e12
    attn_tf = sum(r.attn_flops for r in res) / max(1e-9, sum(r.attn_ms for r in res) / 1e3) / 1e12
    attnb_tf = sum(r.attn_bwd_flops for r in res) / max(1e-9, sum(r.attn_bwd_ms for r in res) / 1e3) / 1e12
    def _tf(f, t):
        return f / max(1e-9, t / 1e3) / 1e12

    def _split(ms_all, fl_all, ms_dep, fl_dep):
        # the class split by chunk kind: dependent chunks (the 37,888-token
        # sequence's pieces, with a KV prefix) vs the packed standalone chunks
        return {"dependent_chunks": {"achieved": _tf(fl_dep, ms_dep), "share_of_step": ms_dep / ms},
                "standalone_chunks": {"achieved": _tf(fl_all - fl_dep, ms_all - ms_dep),
                                      "share_of_step": (ms_all - ms_dep) / ms}}

    attn_split = _split(sum(r.attn_ms for r in res), sum(r.attn_flops for r in res),
                        sum(r.attn_dep_ms for r in res), sum(r.attn_dep_flops for r in res))
    attnb_split = _split(sum(r.attn_bwd_ms for r in res), sum(r.attn_bwd_flops for r in res),
                         sum(r.attn_bwd_dep_ms for r in res), sum(r.attn_bwd_dep_flops for r in res))
    gemm_share = sum(r.gemm_ms for r in res) / ms
    attn_share = sum(r.attn_ms for r in res) / ms
    attnb_share = sum(r.attn_bwd_ms for r in res) / ms
    step_ms = ms_max / args.steps
    value = tokens_all / (step_ms / 1e3)  # tokens of one step over all ranks / slowest rank's step time
    mfu = r0.model_flops * world / (step_ms / 1e3) / 1e12
    cpu = cpu_nproc = c1_gpu = None
    if world == 1 and not args.no_cpu_baseline:
        cpu = cpu_reference_sample(procs=1)
        cpu_nproc = cpu_reference_sample(procs=os.cpu_count() or 1)
        c1_gpu = gpu_c1_side_by_side(ctx)
    line = {
        "metric": METRIC, "value": value, "unit": "tokens/s", "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": step_ms, "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "bf16", "data": "synthetic (SplitMix64 long-tail lengths + tokens, "
                                                      "random-init weights)",
        "config": {"workload": "C2: Llama-7B-shaped (GQA-8) layer stack, 1,000-seq long-tail block per GPU "
                               "(999 log-uniform [16,1024) + 1 x 37,888), chunk 8192, K=1",
                   "global_batch": 1000 * world, "tokens_per_gpu": int(r0.tokens), "chunk_size": CHUNK,
                   "k": K_RETAIN, "parallelism": f"dp{world}",
                   "l2": "inputs larger than L2 (12 GB weights + 25 GB activations per chunk stream through)"},
        "peak_hbm_gb": {"peak": r0.peak_hbm_bytes / 1e9, "static_params_grads": r0.static_hbm_bytes / 1e9,
                        "activations": r0.act_hbm_bytes / 1e9, "kv_state": r0.kv_hbm_bytes / 1e9},
        "mfu": {"model_tflops": mfu, "frac_of_2250": mfu / 2250.0,
                "frac_of_measured_sustained": mfu / pk["bf16_tflops_sustained"]},
        "roofline": {"bound": "tensor", "kernel": "tcgen05 GEMM (all projection/MLP/head GEMMs)",
                     "achieved": gemm_tf, "peak": pk["bf16_tflops_sustained"], "unit": "TFLOP/s",
                     "frac": gemm_tf / pk["bf16_tflops_sustained"], "traffic": traffic[0],
                     "traffic_algorithmic": traffic[1], "traffic_source": TRAFFIC_FILE,
                     "share_of_step": gemm_share, "peak_kind": "measured sustained (MEASURED_PEAKS.json)",
                     "attention_fwd": {"achieved": attn_tf, "share_of_step": attn_share, "unit": "TFLOP/s",
                                       **attn_split},
                     "attention_bwd": {"achieved": attnb_tf, "share_of_step": attnb_share, "unit": "TFLOP/s",
                                       "note": "algorithmic 8*H*dh FLOP/pair", **attnb_split},
                     "other_share_of_step": max(0.0, 1 - gemm_share - attn_share - attnb_share)},
        "hbm_kernels": hbm_kernels(),
        "e2e": {"value": tokens_all / (e2e_max / 1e3 / max(1, args.steps)), "unit": "tokens/s",
                "h2d_bytes_per_step": h2d, "d2h_bytes_per_step": d2h},
        "gpu_launches": int(sum(r.gpu_launches for r in res)),
        "clocks": clk.summary(),
        "loss": r0.loss,
        # run_plan's own instrumentation on the measured step (plan_runner.hpp:36-60)
        "checks": {"recompute_forwards": int(r0.recompute_forward_count),
                   "recompute_loss_mismatches": int(r0.recompute_loss_mismatches),
                   "kv_completeness_violations": int(r0.kv_completeness_violations),
                   "peak_retained_tokens": int(r0.peak_retained_tokens)},
    }
    if cpu:
        line["cpu_baseline"] = {"value": cpu["tokens_per_s"], "unit": "tokens/s", "cores": cpu["cores"],
                                "kind": cpu["kind"], "sample": cpu["sample"]}
        # like-for-like on the C1 workload itself (no FLOP conversion): the
        # reference on 1 core (bounded sample) and on every host core (full
        # batch, disjoint processes) beside the GPU on the full C1 batch
        line["c1_side_by_side"] = {
            "unit": "C1 tokens/s", "workload": "toy V256 d256 H4 KVH2 L2, C1 batch (10,266 tokens), chunk 512, K=2",
            "cpu_reference_1core": cpu["c1_tokens_per_s"], "cpu_reference_all_cores": cpu_nproc["c1_tokens_per_s"],
            "cpu_cores": cpu_nproc["cores"], "gpu_b200": c1_gpu["tokens_per_s"],
            "gpu_note": "plan build + cf_run_plan with host buffers per step; the toy model is launch-bound on a B200"}
    print(json.dumps(line), flush=True)
    if dist:
        dist.destroy_process_group()


# ------------------------------------------------------------- launcher
def _free_port():
    import socket
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def spawn_ranks(args):
    """`python bench.py --gpus N` without torchrun env: re-launch this script
    as N ranks (one process per GPU) with torch.distributed.run on
    127.0.0.1, exactly as the driver does for N > 1, and return its exit code.
    NCCL's communicator-init lines (NCCL_DEBUG=INFO, INIT subsystem) go to
    stderr so the N-rank communicator is visible in the log."""
    env = dict(os.environ)
    if not args.dry_run:
        env.setdefault("NCCL_DEBUG", "INFO")
        env.setdefault("NCCL_DEBUG_SUBSYS", "INIT")
        env.setdefault("NCCL_DEBUG_FILE", "/dev/stderr")
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
           "--master-addr", "127.0.0.1", "--master-port", str(_free_port()), os.path.abspath(__file__)] + sys.argv[1:]
    return subprocess.call(cmd, env=env)


def run_dry(args):
    """CPU rank-wiring check (gloo, no GPU): every rank builds the global
    plan of the N-block batch, takes its DP partition (cf_plan_partition) and
    the global normalizer exactly as run_b200 does; rank 0 verifies that the
    ranks' chunks partition the global plan (each chunk on exactly one rank,
    whole dependent groups together) and prints the bench line's rank fields."""
    import torch
    import torch.distributed as dist
    import paper_2503_02356_b200 as cf

    rank, world, _ = dist_env()
    if world != args.gpus:
        raise SystemExit(f"launched with WORLD_SIZE={world} but --gpus {args.gpus}")
    dist.init_process_group("gloo")
    blocks = [block_lengths(b + 1) for b in range(world)]
    lengths = np.concatenate(blocks)
    ids = np.arange(len(lengths), dtype=np.int64)
    gplan = cf.Plan.build(lengths, CHUNK, K_RETAIN, ids)
    plan = gplan.partition(world, rank) if world > 1 else gplan
    gch = gplan.export()[0]
    ch = plan.export()[0]
    cover = torch.zeros(len(gch), dtype=torch.int64)
    pos = {int(c): i for i, c in enumerate(gch["chunk_id"])}
    for c in ch["chunk_id"]:
        cover[pos[int(c)]] += 1
    grp = torch.full((len(gch),), -1, dtype=torch.int64)
    for c, g in zip(ch["chunk_id"], ch["group_id"]):
        if g >= 0:
            grp[pos[int(c)]] = rank
    dist.all_reduce(cover)
    owners = [torch.zeros_like(grp) for _ in range(world)]
    dist.all_gather(owners, grp)
    tok = torch.tensor([int(ch["total_tokens"].sum())], dtype=torch.int64)
    per_rank = [torch.zeros_like(tok) for _ in range(world)]
    dist.all_gather(per_rank, tok)
    if rank == 0:
        ok = bool((cover == 1).all())
        # every dependent group lives on one rank
        for g in set(int(x) for x in gch["group_id"] if x >= 0):
            rows = [i for i, x in enumerate(gch["group_id"]) if int(x) == g]
            holders = {r for r in range(world) for i in rows if int(owners[r][i]) >= 0}
            ok = ok and len(holders) == 1
        print(json.dumps({"dry_run": True, "metric": METRIC, "value": None, "unit": "tokens/s", "n_gpus": world,
                          "backend": "gloo", "partition_ok": ok,
                          "global_chunks": int(len(gch)), "tokens_per_rank": [int(t.item()) for t in per_rank],
                          "global_tokens": int(lengths.sum()), "normalizer": float((lengths - 1).sum()),
                          "config": {"parallelism": f"dp{world}", "global_batch": 1000 * world}}), flush=True)
    dist.destroy_process_group()


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=3)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="b200", choices=["b200", "reference"])
    ap.add_argument("--workload", default="c2", choices=["c2", "long", "short"],
                    help="c2 = the metric's workload; long/short = slices of it for profiling only")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--dry-run", action="store_true",
                    help="CPU only (gloo): check the N-rank wiring and DP partition, no GPU work")
    args = ap.parse_args()
    global WORKLOAD
    WORKLOAD = args.workload
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        sys.exit(spawn_ranks(args))
    if args.dry_run:
        run_dry(args)
    elif args.impl == "reference":
        run_reference_arm(args)
    else:
        run_b200(args)


if __name__ == "__main__":
    main()
