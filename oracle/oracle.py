"""ctypes front-end for the two CPU checkers — TEST INFRASTRUCTURE ONLY.

* ``Oracle()``    -> oracle/libcforacle.so   (CPU restatement, cf_oracle.cpp)
* ``Reference()`` -> oracle/_ref/libcfref.so (the unmodified reference headers
                     compiled in place by oracle/Makefile)

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / reference
arm may import this module.  The product package never does.
"""
from __future__ import annotations

import ctypes as C
import os

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))

I64 = C.c_int64
PI64 = C.POINTER(C.c_int64)
PD = C.POINTER(C.c_double)
PI32 = C.POINTER(C.c_int32)

CHUNK_DT = np.dtype([(k, np.int64) for k in
                     ("chunk_id", "kind", "group_id", "index_in_group",
                      "total_tokens", "seg_offset", "seg_count")])
SEG_DT = np.dtype([(k, np.int64) for k in ("sequence_id", "start_token", "length")])
EVENT_DT = np.dtype([(k, np.int64) for k in
                     ("kind", "chunk_id", "group_id", "index_in_group",
                      "is_recompute", "save_kv", "read_kv_prefix",
                      "accumulate_kv_grad")])
DIAG_DT = np.dtype([(k, np.int64) for k in
                    ("peak_retained_tokens", "recompute_token_count",
                     "num_violations")])


class ModelCfg(C.Structure):
    _fields_ = [("arch", C.c_int32), ("reserved", C.c_int32),
                ("vocab_size", C.c_int64), ("d_model", C.c_int64),
                ("num_heads", C.c_int64), ("num_kv_heads", C.c_int64),
                ("num_layers", C.c_int64), ("ffn_width", C.c_int64),
                ("seed", C.c_uint64), ("rope_theta", C.c_double),
                ("rms_eps", C.c_double)]


def model_cfg(arch=0, vocab=32, d=16, heads=4, kv_heads=2, layers=2, ffn=0,
              seed=7, rope_theta=10000.0, rms_eps=1e-5) -> ModelCfg:
    return ModelCfg(arch, 0, vocab, d, heads, kv_heads, layers, ffn, seed,
                    rope_theta, rms_eps)


def _p(a, t):
    return a.ctypes.data_as(t)


class _Lib:
    prefix = ""

    def __init__(self, path):
        if not os.path.exists(path):
            raise FileNotFoundError(f"{path} missing: run `make -C oracle`")
        self.lib = C.CDLL(path)
        getattr(self.lib, self.prefix + "last_error").restype = C.c_char_p

    def _fn(self, name):
        return getattr(self.lib, self.prefix + name)

    def _check(self, rc):
        if rc != 0:
            msg = self._fn("last_error")().decode()
            raise ValueError(f"[{rc}] {msg}")

    # -------------------------------------------------------------- planning
    def construct_chunks(self, lengths, chunk_size, ids=None):
        lengths = np.ascontiguousarray(lengths, np.int64)
        ids = np.arange(len(lengths), dtype=np.int64) if ids is None else np.ascontiguousarray(ids, np.int64)
        cap = int(len(lengths) + sum((int(x) + chunk_size - 1) // chunk_size for x in lengths) + 8)
        ch = np.zeros(cap, CHUNK_DT)
        sg = np.zeros(cap, SEG_DT)
        nc, ns = I64(), I64()
        self._check(self._fn("construct_chunks")(
            _p(ids, PI64), _p(lengths, PI64), I64(len(lengths)), I64(chunk_size),
            ch.ctypes.data_as(C.c_void_p), I64(cap), sg.ctypes.data_as(C.c_void_p),
            I64(cap), C.byref(nc), C.byref(ns)))
        return ch[:nc.value].copy(), sg[:ns.value].copy()

    def schedule_step(self, lengths, chunk_size, k, ids=None):
        lengths = np.ascontiguousarray(lengths, np.int64)
        ids = np.arange(len(lengths), dtype=np.int64) if ids is None else np.ascontiguousarray(ids, np.int64)
        cap = int(4 * (len(lengths) + sum((int(x) + chunk_size - 1) // chunk_size for x in lengths)) + 8)
        ev = np.zeros(cap, EVENT_DT)
        dg = np.zeros(1, DIAG_DT)
        ne = I64()
        self._check(self._fn("schedule_step")(
            _p(ids, PI64), _p(lengths, PI64), I64(len(lengths)), I64(chunk_size),
            I64(k), ev.ctypes.data_as(C.c_void_p), I64(cap), C.byref(ne),
            dg.ctypes.data_as(C.c_void_p)))
        return ev[:ne.value].copy(), dg[0]

    def schedule_group(self, n, k, chunk_size=1):
        cap = 4 * n + 8
        ev = np.zeros(cap, EVENT_DT)
        dg = np.zeros(1, DIAG_DT)
        ne = I64()
        self._check(self._fn("schedule_group")(
            I64(n), I64(k), I64(chunk_size), ev.ctypes.data_as(C.c_void_p),
            I64(cap), C.byref(ne), dg.ctypes.data_as(C.c_void_p)))
        return ev[:ne.value].copy(), dg[0]

    def listing(self, lengths, chunk_size, k, ids=None):
        lengths = np.ascontiguousarray(lengths, np.int64)
        ids = np.arange(len(lengths), dtype=np.int64) if ids is None else np.ascontiguousarray(ids, np.int64)
        cap = 64 * (4 * len(lengths) + sum((int(x) + chunk_size - 1) // chunk_size for x in lengths) * 4) + 64
        buf = C.create_string_buffer(cap)
        self._check(self._fn("listing")(_p(ids, PI64), _p(lengths, PI64),
                                        I64(len(lengths)), I64(chunk_size),
                                        I64(k), buf, I64(cap)))
        return buf.value.decode()

    def synthesize(self, count, seed, preset=1, bounds=(), fracs=(), max_length=0):
        b = np.ascontiguousarray(bounds, np.int64)
        f = np.ascontiguousarray(fracs, np.float64)
        out = np.zeros(count, np.int64)
        self._check(self._fn("synthesize")(_p(b, PI64), _p(f, PD), I64(len(b)),
                                           I64(max_length), I64(preset),
                                           I64(count), C.c_uint64(seed),
                                           _p(out, PI64)))
        return out


class Oracle(_Lib):
    """The CPU restatement (oracle/cf_oracle.cpp)."""

    prefix = "cfo_"

    def __init__(self):
        super().__init__(os.path.join(HERE, "libcforacle.so"))
        self.lib.cfo_num_params.restype = C.c_int64
        self.lib.cfo_num_tensors.restype = C.c_int64

    def gen_tokens(self, lengths, vocab, seed):
        lengths = np.ascontiguousarray(lengths, np.int64)
        out = np.zeros(int(lengths.sum()), np.int32)
        self._check(self.lib.cfo_gen_tokens(_p(lengths, PI64), I64(len(lengths)),
                                            I64(vocab), C.c_uint64(seed),
                                            _p(out, PI32)))
        return out

    def shapes(self, cfg):
        n = self.lib.cfo_num_tensors(C.byref(cfg))
        out = []
        for i in range(n):
            r, c = I64(), I64()
            self._check(self.lib.cfo_tensor_shape(C.byref(cfg), I64(i), C.byref(r), C.byref(c)))
            out.append((r.value, c.value))
        return out

    def num_params(self, cfg):
        return self.lib.cfo_num_params(C.byref(cfg))

    def init(self, cfg):
        out = np.zeros(self.num_params(cfg), np.float64)
        self._check(self.lib.cfo_init(C.byref(cfg), _p(out, PD)))
        return out

    def run_plan(self, cfg, lengths, tokens, chunk_size, k, params=None,
                 corrupt=False, normalizer=0.0, ids=None):
        lengths = np.ascontiguousarray(lengths, np.int64)
        ids = np.arange(len(lengths), dtype=np.int64) if ids is None else np.ascontiguousarray(ids, np.int64)
        tokens = np.ascontiguousarray(tokens, np.int32)
        grads = np.zeros(self.num_params(cfg), np.float64)
        loss = C.c_double()
        instr = np.zeros(4, np.int64)
        pp = None if params is None else _p(np.ascontiguousarray(params, np.float64), PD)
        self._check(self.lib.cfo_run_plan(
            C.byref(cfg), pp, _p(ids, PI64), _p(lengths, PI64), _p(tokens, PI32),
            I64(len(lengths)), I64(chunk_size), I64(k), C.c_int(int(corrupt)),
            C.c_double(normalizer), C.byref(loss), _p(grads, PD), _p(instr, PI64)))
        return loss.value, grads, instr

    def backward_full(self, cfg, lengths, tokens, params=None, normalizer=0.0, ids=None):
        lengths = np.ascontiguousarray(lengths, np.int64)
        ids = np.arange(len(lengths), dtype=np.int64) if ids is None else np.ascontiguousarray(ids, np.int64)
        tokens = np.ascontiguousarray(tokens, np.int32)
        grads = np.zeros(self.num_params(cfg), np.float64)
        loss = C.c_double()
        pp = None if params is None else _p(np.ascontiguousarray(params, np.float64), PD)
        self._check(self.lib.cfo_backward_full(
            C.byref(cfg), pp, _p(ids, PI64), _p(lengths, PI64), _p(tokens, PI32),
            I64(len(lengths)), C.c_double(normalizer), C.byref(loss), _p(grads, PD)))
        return loss.value, grads

    def forward_full(self, cfg, lengths, tokens, params=None, normalizer=0.0, ids=None):
        lengths = np.ascontiguousarray(lengths, np.int64)
        ids = np.arange(len(lengths), dtype=np.int64) if ids is None else np.ascontiguousarray(ids, np.int64)
        tokens = np.ascontiguousarray(tokens, np.int32)
        loss = C.c_double()
        pp = None if params is None else _p(np.ascontiguousarray(params, np.float64), PD)
        self._check(self.lib.cfo_forward_full(
            C.byref(cfg), pp, _p(ids, PI64), _p(lengths, PI64), _p(tokens, PI32),
            I64(len(lengths)), C.c_double(normalizer), C.byref(loss)))
        return loss.value


class Reference(_Lib):
    """The unmodified reference, compiled in place (oracle/_ref/libcfref.so)."""

    prefix = "cfr_"

    def __init__(self):
        super().__init__(os.path.join(HERE, "_ref", "libcfref.so"))
        self.lib.cfr_toy_num_params.restype = C.c_int64
        self.lib.cfr_last_error.restype = C.c_char_p

    def num_params(self, cfg):
        return self.lib.cfr_toy_num_params(C.byref(cfg))

    def init(self, cfg):
        out = np.zeros(self.num_params(cfg), np.float64)
        self._check(self.lib.cfr_toy_init(C.byref(cfg), _p(out, PD)))
        return out

    def run_plan(self, cfg, lengths, tokens, chunk_size, k, corrupt=False, ids=None):
        lengths = np.ascontiguousarray(lengths, np.int64)
        ids = np.arange(len(lengths), dtype=np.int64) if ids is None else np.ascontiguousarray(ids, np.int64)
        tokens = np.ascontiguousarray(tokens, np.int32)
        grads = np.zeros(self.num_params(cfg), np.float64)
        loss = C.c_double()
        instr = np.zeros(4, np.int64)
        self._check(self.lib.cfr_run_plan(
            C.byref(cfg), _p(ids, PI64), _p(lengths, PI64), _p(tokens, PI32),
            I64(len(lengths)), I64(chunk_size), I64(k), C.c_int(int(corrupt)),
            C.byref(loss), _p(grads, PD), _p(instr, PI64)))
        return loss.value, grads, instr

    def backward_full(self, cfg, lengths, tokens, ids=None):
        lengths = np.ascontiguousarray(lengths, np.int64)
        ids = np.arange(len(lengths), dtype=np.int64) if ids is None else np.ascontiguousarray(ids, np.int64)
        tokens = np.ascontiguousarray(tokens, np.int32)
        grads = np.zeros(self.num_params(cfg), np.float64)
        loss = C.c_double()
        self._check(self.lib.cfr_backward_full(
            C.byref(cfg), _p(ids, PI64), _p(lengths, PI64), _p(tokens, PI32),
            I64(len(lengths)), C.byref(loss), _p(grads, PD)))
        return loss.value, grads

    def simulate(self, lengths, chunk_size, k, stages, alpha=1.0, beta=0.0,
                 gamma=0.0, hop=0.0, mode=1, ids=None):
        lengths = np.ascontiguousarray(lengths, np.int64)
        ids = np.arange(len(lengths), dtype=np.int64) if ids is None else np.ascontiguousarray(ids, np.int64)
        mk, bb = C.c_double(), C.c_double()
        self._check(self.lib.cfr_simulate(
            _p(ids, PI64), _p(lengths, PI64), I64(len(lengths)), I64(chunk_size),
            I64(k), I64(stages), C.c_double(alpha), C.c_double(beta),
            C.c_double(gamma), C.c_double(hop), C.c_int(mode), C.byref(mk),
            C.byref(bb)))
        return mk.value, bb.value


    def pp_trace(self, lengths, chunk_size, k, stages, cost=(0.0, 1.0, 0.0, 2.0, 0.0), mode=1,
                 backward_first=True, ids=None):
        """Full reference trace: (ops[stages, per, 4] = kind, chunk, start, end;
        busy; busy_total; makespan; bubble)."""
        lengths = np.ascontiguousarray(lengths, np.int64)
        ids = np.arange(len(lengths), dtype=np.int64) if ids is None else np.ascontiguousarray(ids, np.int64)
        c5 = np.ascontiguousarray(cost, np.float64)
        per, mk, bb = C.c_int64(), C.c_double(), C.c_double()
        args = lambda ops, busy, busy_t: (  # noqa: E731
            _p(ids, PI64), _p(lengths, PI64), I64(len(lengths)), I64(chunk_size), I64(k), I64(stages),
            _p(c5, PD), C.c_int(mode), C.c_int(int(backward_first)), ops, C.byref(per), busy, busy_t,
            C.byref(mk), C.byref(bb))
        self._check(self.lib.cfr_pp_trace(*args(None, None, None)))
        ops = np.zeros((stages, per.value, 4), np.float64)
        busy = np.zeros(stages, np.float64)
        busy_t = np.zeros(stages, np.float64)
        self._check(self.lib.cfr_pp_trace(*args(_p(ops, PD), _p(busy, PD), _p(busy_t, PD))))
        return ops, busy, busy_t, mk.value, bb.value


    def _text(self, call):
        n = C.c_size_t()
        self._check(call(None, C.c_size_t(0), C.byref(n)))
        buf = C.create_string_buffer(n.value + 1)
        self._check(call(buf, C.c_size_t(n.value + 1), C.byref(n)))
        return buf.raw[:n.value].decode()

    def plan_json(self, lengths, chunk_size, k=1, which=0, ids=None):
        lengths = np.ascontiguousarray(lengths, np.int64)
        ids = np.arange(len(lengths), dtype=np.int64) if ids is None else np.ascontiguousarray(ids, np.int64)
        return self._text(lambda b, c, n: self.lib.cfr_plan_json(
            _p(ids, PI64), _p(lengths, PI64), I64(len(lengths)), I64(chunk_size), I64(k), C.c_int(which), b, c, n))

    def schedule_json(self, doc: str, k):
        return self._text(lambda b, c, n: self.lib.cfr_schedule_json(doc.encode(), I64(k), b, c, n))

    def jsonl_roundtrip(self, text: str):
        return self._text(lambda b, c, n: self.lib.cfr_jsonl_roundtrip(text.encode(), b, c, n))

    def calibrate(self, csv: str, gqa=1.0):
        coeffs = np.zeros(4, np.float64)
        res = C.c_double()
        doc = self._text(lambda b, c, n: self.lib.cfr_calibrate(csv.encode(), C.c_double(gqa), _p(coeffs, PD),
                                                               C.byref(res), b, c, n))
        return coeffs, res.value, doc


    def export_trace(self, lengths, chunk_size, k, stages, cost=(0.0, 1.0, 0.0, 2.0, 0.0), mode=1, chrome=True):
        lengths = np.ascontiguousarray(lengths, np.int64)
        ids = np.arange(len(lengths), dtype=np.int64)
        c5 = np.ascontiguousarray(cost, np.float64)
        return self._text(lambda b, c, n: self.lib.cfr_export_trace(
            _p(ids, PI64), _p(lengths, PI64), I64(len(lengths)), I64(chunk_size), I64(k), I64(stages), _p(c5, PD),
            C.c_int(mode), C.c_int(0 if chrome else 1), b, c, n))


    def tune(self, lengths, css, ks, stages, cost, mem, budget, gbs, nb, seed, csv=True, ids=None):
        lengths = np.ascontiguousarray(lengths, np.int64)
        ids = np.arange(len(lengths), dtype=np.int64) if ids is None else np.ascontiguousarray(ids, np.int64)
        css = np.ascontiguousarray(css, np.int64)
        ks = np.ascontiguousarray(ks, np.int64)
        c5 = np.ascontiguousarray(cost, np.float64)
        m4 = np.ascontiguousarray(mem, np.float64)
        return self._text(lambda b, c, n: self.lib.cfr_tune(
            _p(ids, PI64), _p(lengths, PI64), I64(len(lengths)), _p(css, PI64), I64(len(css)), _p(ks, PI64),
            I64(len(ks)), I64(stages), _p(c5, PD), _p(m4, PD), C.c_double(budget), I64(gbs), I64(nb),
            C.c_uint64(seed), C.c_int(int(csv)), b, c, n))


def c1_batch(oracle: Oracle):
    """Config C1 canonical batch: synthesize(eval_table5, 32,
    seed=3) plus sequence id 32 of 2048 tokens; tokens SplitMix64(5)."""
    lengths = list(oracle.synthesize(32, 3, preset=1)) + [2048]
    lengths = np.asarray(lengths, np.int64)
    tokens = oracle.gen_tokens(lengths, 256, 5)
    return lengths, tokens


def c1_cfg(arch=0):
    return model_cfg(arch=arch, vocab=256, d=256, heads=4, kv_heads=2, layers=2,
                     ffn=0 if arch == 0 else 512, seed=1)
