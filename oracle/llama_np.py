"""Vectorised fp64 restatement of forward_full / backward_full — TEST
INFRASTRUCTURE ONLY (same import rules as oracle/oracle.py: tests/,
__graft_entry__.smoke() and bench.py's CPU legs only; the product never
imports it).

Why a second restatement: the C++ oracle (cf_oracle.cpp) follows the
reference's row-by-row GEMV structure (toy_model.hpp:166-198) and runs at
~20 GFLOP/s, which is fine up to d = 256 but needs tens of minutes for a
production-width (d 4096, ffn 11008, V 32000) layer.  This module computes the
same per-sequence unchunked step with BLAS GEMMs (~1 TFLOP/s fp64), so the
GPU's chunked run_plan can be compared with an fp64 oracle at the shapes the
B200 path actually runs (the verify_equivalence comparison,
plan_runner.hpp:368-395: chunked run vs backward_full).

Parity of this restatement is pinned against the C++ oracle — itself bitwise
equal to the compiled reference on the toy arch — in
tests/test_oracle_pinning.py (loss and every gradient to 1e-12 relative; the
summation order differs, so bitwise equality is not expected).

Semantics followed (file:line under /root/reference/proj/include/chunkflow/):
* tensor order and [in, out] layout: toy_model.hpp:116-126 (+ the llama
  extension of cf_oracle.cpp: attn_norm, wq, wk, wv, wo, ffn_norm, w_gate,
  w_up, w_down per layer; final_norm before head);
* forward: toy_model.hpp:206-334 (embedding, per-layer QKV, causal GQA
  attention with scale 1/sqrt(dh) and kv head = hq // (H / KVH), Wo +
  residual, FFN + residual, CE over positions with a target);
* backward: toy_model.hpp:341-520; the embedding gradient scatters per token;
* backward_full: toy_model.hpp:575-596 — every sequence alone, one global
  normalizer sum(len - 1) (toy_model.hpp:533-541).
Llama extension (no reference exists; as cf_oracle.cpp): RMSNorm
y = x * rsqrt(mean(x^2) + eps) * g, rotate-half RoPE at absolute positions
with inv_freq = theta^(-2i/dh), SwiGLU h = silu(gate) * up.
"""
from __future__ import annotations

import numpy as np


class Shapes:
    def __init__(self, cfg):
        self.arch = int(cfg.arch)
        self.V = int(cfg.vocab_size)
        self.d = int(cfg.d_model)
        self.H = int(cfg.num_heads)
        self.KVH = int(cfg.num_kv_heads)
        self.L = int(cfg.num_layers)
        self.llama = self.arch == 1
        self.ffn = int(cfg.ffn_width) if self.llama else 2 * self.d
        self.dh = self.d // self.H
        self.kvw = self.KVH * self.dh
        self.theta = float(cfg.rope_theta)
        self.eps = float(cfg.rms_eps)

    def tensors(self):
        d, kvw, f = self.d, self.kvw, self.ffn
        out = [("embedding", self.V, d)]
        for l in range(self.L):
            p = f"layer{l}."
            if self.llama:
                out += [(p + "attn_norm", 1, d), (p + "wq", d, d), (p + "wk", d, kvw), (p + "wv", d, kvw),
                        (p + "wo", d, d), (p + "ffn_norm", 1, d), (p + "w_gate", d, f), (p + "w_up", d, f),
                        (p + "w_down", f, d)]
            else:
                out += [(p + "wq", d, d), (p + "wk", d, kvw), (p + "wv", d, kvw), (p + "wo", d, d),
                        (p + "w1", d, f), (p + "w2", f, d)]
        if self.llama:
            out.append(("final_norm", 1, d))
        out.append(("head", d, self.V))
        return out


def _views(flat, shapes):
    """name -> [rows, cols] view into the flat parameter (or gradient) vector."""
    out, off = {}, 0
    for name, r, c in shapes.tensors():
        out[name] = flat[off:off + r * c].reshape(r, c)
        off += r * c
    assert off == flat.size, (off, flat.size)
    return out


def _rope_tables(s, T):
    half = s.dh // 2
    i = np.arange(half, dtype=np.float64)
    f = np.power(s.theta, -2.0 * i / float(s.dh))
    a = np.arange(T, dtype=np.float64)[:, None] * f[None, :]
    return np.cos(a), np.sin(a)


def _rope(x, heads, dh, cos, sin, inverse=False):
    """rotate-half on [T, heads*dh] (cf_oracle.cpp rope())."""
    T = x.shape[0]
    v = x.reshape(T, heads, dh)
    half = dh // 2
    x0, x1 = v[:, :, :half].copy(), v[:, :, half:].copy()
    c, s_ = cos[:, None, :], (-sin if inverse else sin)[:, None, :]
    out = np.empty_like(v)
    out[:, :, :half] = x0 * c - x1 * s_
    out[:, :, half:] = x1 * c + x0 * s_
    return out.reshape(T, heads * dh)


def _rms(x, g, eps):
    r = 1.0 / np.sqrt((x * x).mean(axis=1) + eps)
    return x * r[:, None] * g[None, :], r


def _rms_bwd(x, g, r, dy):
    """(dx, dgain) of y = x * r * g (cf_oracle.cpp rms_bwd)."""
    d = x.shape[1]
    dot = (dy * g[None, :] * x).sum(axis=1)
    k = r ** 3 * dot / d
    dx = r[:, None] * dy * g[None, :] - x * k[:, None]
    dg = (dy * x * r[:, None]).sum(axis=0)
    return dx, dg


def _sigm(x):
    return 1.0 / (1.0 + np.exp(-x))


def _seq_step(s, P, G, tok, norm, want_grad):
    """Forward (+ backward into G) of one whole sequence; returns loss_sum."""
    T, d, H, KVH, dh, kvw = tok.size, s.d, s.H, s.KVH, s.dh, s.kvw
    per = H // KVH
    inv = 1.0 / np.sqrt(float(dh))
    cos, sin = _rope_tables(s, T) if s.llama else (None, None)
    causal = np.tril(np.ones((T, T), dtype=bool))
    x = P["embedding"][tok].astype(np.float64)
    tapes = []
    for l in range(s.L):
        p = f"layer{l}."
        tp = {"x_in": x}
        if s.llama:
            xn, r1 = _rms(x, P[p + "attn_norm"][0], s.eps)
            tp["r1"] = r1
        else:
            xn = x
        tp["xn"] = xn
        q = xn @ P[p + "wq"]
        k = xn @ P[p + "wk"]
        v = xn @ P[p + "wv"]
        if s.llama:
            q = _rope(q, H, dh, cos, sin)
            k = _rope(k, KVH, dh, cos, sin)
        attn = np.empty((T, d))
        probs = []
        for g in range(KVH):
            kg = k[:, g * dh:(g + 1) * dh]
            vg = v[:, g * dh:(g + 1) * dh]
            qg = q[:, g * per * dh:(g + 1) * per * dh].reshape(T, per, dh).transpose(1, 0, 2)  # [per,T,dh]
            sc = (qg @ kg.T) * inv
            sc = np.where(causal[None], sc, -np.inf)
            sc -= sc.max(axis=2, keepdims=True)
            e = np.exp(sc)
            pr = e / e.sum(axis=2, keepdims=True)
            og = pr @ vg  # [per,T,dh]
            attn[:, g * per * dh:(g + 1) * per * dh] = og.transpose(1, 0, 2).reshape(T, per * dh)
            probs.append(pr if want_grad else None)
        tp.update(q=q, k=k, v=v, attn=attn, probs=probs)
        mid = attn @ P[p + "wo"] + x
        tp["mid"] = mid
        if s.llama:
            xn2, r2 = _rms(mid, P[p + "ffn_norm"][0], s.eps)
            gt = xn2 @ P[p + "w_gate"]
            up = xn2 @ P[p + "w_up"]
            h = gt * _sigm(gt) * up
            x = h @ P[p + "w_down"] + mid
            tp.update(xn2=xn2, r2=r2, gt=gt, up=up, h=h)
        else:
            h = np.tanh(mid @ P[p + "w1"])
            x = h @ P[p + "w2"] + mid
            tp["h"] = h
        tapes.append(tp)
    if s.llama:
        xf, rf = _rms(x, P["final_norm"][0], s.eps)
    else:
        xf, rf = x, None
    tgt = tok[1:]
    logits = xf[:-1] @ P["head"]  # positions with a target: 0..T-2
    mx = logits.max(axis=1, keepdims=True)
    e = np.exp(logits - mx)
    den = e.sum(axis=1, keepdims=True)
    lse = (mx + np.log(den))[:, 0]
    loss_sum = float((lse - logits[np.arange(T - 1), tgt]).sum())
    if not want_grad:
        return loss_sum
    dl = e / den
    dl[np.arange(T - 1), tgt] -= 1.0
    dl /= norm
    G["head"] += xf[:-1].T @ dl
    dxf = np.zeros((T, d))
    dxf[:-1] = dl @ P["head"].T
    del dl, e, logits
    if s.llama:
        dx, dgf = _rms_bwd(x, P["final_norm"][0], rf, dxf)
        G["final_norm"][0] += dgf
    else:
        dx = dxf
    for l in reversed(range(s.L)):
        p = f"layer{l}."
        tp = tapes[l]
        if s.llama:
            dh_ = dx @ P[p + "w_down"].T
            G[p + "w_down"] += tp["h"].T @ dx
            sg = _sigm(tp["gt"])
            du = dh_ * tp["gt"] * sg
            dg_ = dh_ * tp["up"] * sg * (1.0 + tp["gt"] * (1.0 - sg))
            dxn2 = dg_ @ P[p + "w_gate"].T + du @ P[p + "w_up"].T
            G[p + "w_gate"] += tp["xn2"].T @ dg_
            G[p + "w_up"] += tp["xn2"].T @ du
            ddm, dg2 = _rms_bwd(tp["mid"], P[p + "ffn_norm"][0], tp["r2"], dxn2)
            G[p + "ffn_norm"][0] += dg2
            dmid = dx + ddm
        else:
            da = (dx @ P[p + "w2"].T) * (1.0 - tp["h"] ** 2)
            G[p + "w2"] += tp["h"].T @ dx
            dmid = dx + da @ P[p + "w1"].T
            G[p + "w1"] += tp["mid"].T @ da
        dattn = dmid @ P[p + "wo"].T
        G[p + "wo"] += tp["attn"].T @ dmid
        q, k, v = tp["q"], tp["k"], tp["v"]
        dq = np.empty((T, d))
        dk = np.zeros((T, kvw))
        dv = np.zeros((T, kvw))
        for g in range(KVH):
            pr = tp["probs"][g]  # [per,T,T]
            kg = k[:, g * dh:(g + 1) * dh]
            vg = v[:, g * dh:(g + 1) * dh]
            qg = q[:, g * per * dh:(g + 1) * per * dh].reshape(T, per, dh).transpose(1, 0, 2)
            dog = dattn[:, g * per * dh:(g + 1) * per * dh].reshape(T, per, dh).transpose(1, 0, 2)
            dp = dog @ vg.T
            ds = pr * (dp - (pr * dp).sum(axis=2, keepdims=True)) * inv
            dq[:, g * per * dh:(g + 1) * per * dh] = (ds @ kg).transpose(1, 0, 2).reshape(T, per * dh)
            dk[:, g * dh:(g + 1) * dh] = np.einsum("pts,ptu->su", ds, qg)
            dv[:, g * dh:(g + 1) * dh] = np.einsum("pts,ptu->su", pr, dog)
        if s.llama:
            dq = _rope(dq, H, dh, cos, sin, inverse=True)
            dk = _rope(dk, KVH, dh, cos, sin, inverse=True)
        xn = tp["xn"]
        G[p + "wq"] += xn.T @ dq
        G[p + "wk"] += xn.T @ dk
        G[p + "wv"] += xn.T @ dv
        dxn = dq @ P[p + "wq"].T + dk @ P[p + "wk"].T + dv @ P[p + "wv"].T
        if s.llama:
            ddx, dg1 = _rms_bwd(tp["x_in"], P[p + "attn_norm"][0], tp["r1"], dxn)
            G[p + "attn_norm"][0] += dg1
            dx = dmid + ddx
        else:
            dx = dmid + dxn
        tapes[l] = None
    np.add.at(G["embedding"], tok, dx)
    return loss_sum


def backward_full(cfg, params, lengths, tokens, normalizer=0.0):
    """(loss, flat fp64 gradients) of the unchunked batch (toy_model.hpp:575):
    every sequence alone, loss = sum of per-sequence CE sums / normalizer."""
    s = Shapes(cfg)
    params = np.ascontiguousarray(params, np.float64)
    P = _views(params, s)
    grads = np.zeros_like(params)
    G = _views(grads, s)
    lengths = np.asarray(lengths, np.int64)
    norm = float(normalizer) if normalizer > 0 else float((lengths - 1).sum())
    off, total = 0, 0.0
    for n in lengths:
        tok = np.asarray(tokens[off:off + n], np.int64)
        off += int(n)
        total += _seq_step(s, P, G, tok, norm, True)
    return total / norm, grads


def forward_full(cfg, params, lengths, tokens, normalizer=0.0):
    s = Shapes(cfg)
    P = _views(np.ascontiguousarray(params, np.float64), s)
    lengths = np.asarray(lengths, np.int64)
    norm = float(normalizer) if normalizer > 0 else float((lengths - 1).sum())
    off, total = 0, 0.0
    for n in lengths:
        tok = np.asarray(tokens[off:off + n], np.int64)
        off += int(n)
        total += _seq_step(s, P, None, tok, norm, False)
    return total / norm
