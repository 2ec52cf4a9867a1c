"""The persistent attention kernels (attn_fwd_pp_persist_kernel,
attention_tc_fwd2.cu; dkv_persist_kernel, attention_tc_bwd.cu) against the
one-CTA-per-item kernels they restructure.  The choice is read from
CF_FWD_PERSIST / CF_DKV_PERSIST once per process, so each variant runs in a
child process on the same seeded inputs and the outputs must be bitwise equal
(same per-item arithmetic order): operator-level forward and backward, and
the parameter gradients of a run_plan step (standalone chunks take the
direct bf16 dK/dV read-out, the dependent group the fp32 accumulators).  The
persistent kernels' numerics are checked against the fp32 reference by
test_attention_gpu.py (they are the default); the per-item kernels keep that
suite in a child."""
import os
import subprocess
import sys

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)

# packed short sequences (many items per CTA, ragged tiles, a 1-token
# segment) plus a dependent segment with a KV prefix; 8 q heads / 2 kv heads
_CHILD = r"""
import sys, numpy as np, torch
sys.path.insert(0, {root!r})
import paper_2503_02356_b200 as cf
H, KVH, dh = 8, 2, 128
lens = [700, 1, 33, 128, 129, 5, 300, 64, 250, 17, 90, 511, 40]
segs, q0 = [], 0
for L in lens:
    segs.append((q0, L, q0, 0)); q0 += L
T = q0
segs.append((T, 300, T, 600))  # dependent: keys [T, T + 900), 600 of them prefix
T += 300
R = T + 600
g = torch.Generator(device="cuda").manual_seed(5)
q = torch.randn(T, H * dh, generator=g, device="cuda").to(torch.bfloat16)
k = torch.randn(R, KVH * dh, generator=g, device="cuda").to(torch.bfloat16)
v = torch.randn(R, KVH * dh, generator=g, device="cuda").to(torch.bfloat16)
o = torch.full((T, H * dh), 7.0, device="cuda", dtype=torch.bfloat16)
lse = torch.zeros(H, T, device="cuda")
ctx = cf.Context(0)
ctx.attention(3, False, q.data_ptr(), H * dh, k.data_ptr(), v.data_ptr(), KVH * dh, R, o.data_ptr(),
              lse.data_ptr(), 0, 0, 0, 0, 0, segs, T, H, KVH, dh)
torch.cuda.synchronize()
np.save({out!r} + "_o.npy", o.view(torch.int16).cpu().numpy())
np.save({out!r} + "_lse.npy", lse.cpu().numpy())
dout = torch.randn(T, H * dh, generator=g, device="cuda").to(torch.bfloat16)
dq = torch.zeros(T, H * dh, device="cuda", dtype=torch.bfloat16)
dk = torch.zeros(R, KVH * dh, device="cuda")
dv = torch.zeros(R, KVH * dh, device="cuda")
ctx.attention(1, True, q.data_ptr(), H * dh, k.data_ptr(), v.data_ptr(), KVH * dh, R, o.data_ptr(),
              lse.data_ptr(), dout.data_ptr(), dq.data_ptr(), dk.data_ptr(), dv.data_ptr(), KVH * dh, segs, T, H,
              KVH, dh)
torch.cuda.synchronize()
np.save({out!r} + "_dq.npy", dq.view(torch.int16).cpu().numpy())
np.save({out!r} + "_dk.npy", dk.cpu().numpy())
np.save({out!r} + "_dv.npy", dv.cpu().numpy())
# a run_plan step: packed standalone chunks + a dependent group
cfg = cf.model_cfg(arch=cf.ARCH_LLAMA, vocab=96, d=256, heads=2, kv_heads=1, layers=2, ffn=512, seed=7)
lengths = np.array([8, 30, 64, 300, 33, 200, 129], np.int64)
tokens = cf.gen_tokens(lengths, 96, 11)
model = cf.Model(ctx, cfg)
r = model.run_plan(cf.Plan.build(lengths, 192, 1), lengths, tokens)
np.save({out!r} + "_grads.npy", model.grads_flat())
np.save({out!r} + "_loss.npy", np.array([r.loss]))
"""


_NAMES = ("o", "lse", "dq", "dk", "dv", "grads", "loss")


def _run(tmp_path, persist):
    out = str(tmp_path / f"v{persist}")
    env = dict(os.environ, CF_FWD_PERSIST=str(persist), CF_DKV_PERSIST=str(persist))
    r = subprocess.run([sys.executable, "-c", _CHILD.format(root=ROOT, out=out)], cwd=ROOT, env=env,
                       capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stdout[-2000:] + r.stderr[-2000:]
    return {n: np.load(out + f"_{n}.npy") for n in _NAMES}


def test_persistent_kernels_bitwise_equal_per_item_kernels(tmp_path):
    p, q = _run(tmp_path, 1), _run(tmp_path, 0)
    for n in _NAMES:
        a, b = p[n], q[n]
        if a.dtype.kind == "f":  # compare bit patterns
            bits = np.int32 if a.dtype == np.float32 else np.int64
            a, b = a.view(bits), b.view(bits)
        assert np.array_equal(a, b), n
    assert not np.all(p["o"] == p["o"].flat[0])  # outputs were written
    assert np.abs(p["dk"]).max() > 0 and np.abs(p["grads"]).max() > 0


def test_per_item_kernels_pass_the_attention_suite():
    env = dict(os.environ, CF_FWD_PERSIST="0", CF_DKV_PERSIST="0")
    r = subprocess.run([sys.executable, "-m", "pytest", "-q", "-x", "-m", "gpu", "-p", "no:cacheprovider",
                        os.path.join(HERE, "test_attention_gpu.py")],
                       cwd=ROOT, env=env, capture_output=True, text=True, timeout=900)
    assert r.returncode == 0, r.stdout[-3000:] + r.stderr[-2000:]
    assert " passed" in r.stdout
