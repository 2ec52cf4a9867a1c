"""B200-native ChunkFlow training path (arXiv 2503.02356).

Host planning (chunk construction, state-aware scheduling, DP partition) is
C++; the chunk forward/backward is hand-written sm_100a CUDA; both live in
libchunkflow_b200.so behind the C-ABI in include/chunkflow_b200.h.  This
package is the thin Python face of that library (ctypes), mirroring the
reference's chunkflow:: API names for tests and benchmarks.
"""
from .capi import (ARCH_LLAMA, ARCH_TOY, Context, Model, ModelCfg, Plan, RunResult,  # noqa: F401
                   Step, gen_tokens, lib)
from .api import (construct_chunks, schedule_step, validate_plan, run_plan,  # noqa: F401
                  verify_equivalence, compare_gradients, model_cfg)

__all__ = ["Context", "Model", "ModelCfg", "Plan", "Step", "RunResult", "gen_tokens",
           "construct_chunks", "schedule_step", "validate_plan", "run_plan",
           "verify_equivalence", "compare_gradients", "model_cfg", "lib",
           "ARCH_TOY", "ARCH_LLAMA"]
