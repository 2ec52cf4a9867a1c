"""Config C3 (BASELINE.json): Llama-7B-shaped model, chunk 8192, K=2, the
C2 long-tail block with its long sequence set to 16K / 32K / 64K / 128K.
Reports peak HBM per point, decomposed into static (params + fp32 grads),
retained activations (<= K chunk tapes) and per-sequence KV state, plus
tokens/s.  Peak activations must stay flat in the max sequence length;
only the KV-state term grows."""
import json
import sys
import time

import numpy as np
import torch

sys.path.insert(0, ".")
import paper_2503_02356_b200 as cf  # noqa: E402

MODEL = dict(vocab=32000, d=4096, heads=32, kv_heads=8, layers=32, ffn=11008, seed=1)
ctx = cf.Context(0)
model = cf.Model(ctx, cf.model_cfg(arch=cf.ARCH_LLAMA, **MODEL))
short = cf.capi.synthesize(999, 1, preset=0, bounds=[1024], fracs=[1.0], max_length=1024)
# --offload: dependent groups keep their KV state in pinned host memory
# (cf_run_opts.kv_offload), so the one term that grows with the sequence
# leaves HBM too
offload = "--offload" in sys.argv
sizes = [int(x) for x in sys.argv[1:] if not x.startswith("--")] or [16384, 32768, 65536, 131072]
for L in sizes:
    lengths = np.concatenate([short, [L]]).astype(np.int64)
    tokens = cf.gen_tokens(lengths, MODEL["vocab"], 1)
    plan = cf.Plan.build(lengths, 8192, 2)
    step = cf.Step(model, plan, lengths, tokens)
    step.run(kv_offload=offload)  # warm-up
    ctx.synchronize()
    t0 = time.perf_counter()
    r = step.run(kv_offload=offload)
    ctx.synchronize()
    dt = time.perf_counter() - t0
    free, total = torch.cuda.mem_get_info()
    nc, _, ne, _ = plan.counts()
    print(json.dumps({
        "max_seq": L, "kv_offload": offload, "chunks": nc, "events": ne, "tokens": int(r.tokens), "step_s": dt,
        "tokens_per_s": r.tokens / dt, "loss": r.loss,
        "peak_hbm_gb": r.peak_hbm_bytes / 1e9, "static_gb": r.static_hbm_bytes / 1e9,
        "activations_gb": r.act_hbm_bytes / 1e9, "kv_state_gb": r.kv_hbm_bytes / 1e9,
        "peak_retained_tokens": int(r.peak_retained_tokens), "recompute_forwards": int(r.recompute_forward_count),
        "device_used_gb_after": (total - free) / 1e9}), flush=True)
    step.close()
