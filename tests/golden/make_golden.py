"""Generates tests/golden/*.json from the UNMODIFIED reference, compiled in
place from /root/reference by oracle/Makefile (oracle/_ref/libcfref.so).

Run here (the reference tree does not exist on the GPU box):
    make -C oracle && python tests/golden/make_golden.py
The fixtures are small and committed; tests on any machine compare both the
CPU oracle and the B200 product against them.
"""
import json
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
from oracle.oracle import Reference, c1_cfg, model_cfg  # noqa: E402

OUT = os.path.dirname(os.path.abspath(__file__))


def plan_doc(ref, lengths, cs, k):
    ch, sg = ref.construct_chunks(lengths, cs)
    ev, dg = ref.schedule_step(lengths, cs, k)
    return {"lengths": [int(x) for x in lengths], "chunk_size": cs, "k": k,
            "chunks": ch.tolist(), "segments": sg.tolist(), "events": ev.tolist(),
            "diag": [int(x) for x in dg.tolist()],
            "listing": ref.listing(lengths, cs, k)}


def splitmix_tokens(lengths, vocab, seed):
    # SplitMix64(seed).next_below(vocab) per token (chunkflow_main.cpp:427-443)
    mask = (1 << 64) - 1
    s = seed
    out = []
    thr = ((1 << 64) - vocab) % vocab
    for n in lengths:
        for _ in range(int(n)):
            while True:
                s = (s + 0x9E3779B97F4A7C15) & mask
                z = s
                z = ((z ^ (z >> 30)) * 0xBF58476D1CE4E5B9) & mask
                z = ((z ^ (z >> 27)) * 0x94D049BB133111EB) & mask
                z ^= z >> 31
                if z >= thr:
                    out.append(z % vocab)
                    break
    return np.array(out, np.int32)


def main():
    ref = Reference()
    docs = {}
    # worked batch [1,1,2,4] (test_chunker.cpp / test_scheduler.cpp)
    docs["worked_cs2_k1"] = plan_doc(ref, [1, 1, 2, 4], 2, 1)
    docs["worked_cs4_k1"] = plan_doc(ref, [1, 1, 2, 4], 4, 1)
    docs["ffd_beaten_cs10"] = plan_doc(ref, [5, 4, 4, 3, 2, 2], 10, 1)
    rng = np.random.default_rng(2024)
    docs["random"] = []
    for _ in range(60):
        n = int(rng.integers(1, 40))
        cs = int(rng.integers(2, 64))
        k = int(rng.integers(1, 5))
        lengths = rng.integers(1, 200, n)
        docs["random"].append(plan_doc(ref, lengths, cs, k))
    # C1 canonical batch + the reference's run_plan on it
    lengths = list(ref.synthesize(32, 3, preset=1)) + [2048]
    docs["c1_plan"] = plan_doc(ref, lengths, 512, 2)
    cfg = c1_cfg()
    tokens = splitmix_tokens(lengths, 256, 5)
    loss, grads, instr = ref.run_plan(cfg, lengths, tokens, 512, 2)
    head = grads[-256 * 256:]
    docs["c1_run"] = {"loss": loss, "grad_sum": float(grads.sum()), "grad_abs_sum": float(np.abs(grads).sum()),
                      "head_grad_00_02": [float(x) for x in head[:3]], "instr": [int(x) for x in instr],
                      "token_head": [int(x) for x in tokens[:16]], "token_sum": int(tokens.sum())}
    # verify-CLI defaults (chunkflow_main.cpp:230-245)
    v_len = [8, 8, 16, 32]
    v_tok = splitmix_tokens(v_len, 32, 11)
    vcfg = model_cfg()
    l, g, i = ref.run_plan(vcfg, v_len, v_tok, 16, 1)
    lf, gf = ref.backward_full(vcfg, v_len, v_tok)
    docs["verify_defaults"] = {"lengths": v_len, "tokens": v_tok.tolist(), "loss": l, "loss_full": lf,
                               "grads": g.tolist(), "grads_full": gf.tolist(), "instr": [int(x) for x in i],
                               "params": ref.init(vcfg).tolist()}
    # C2 / C4 batch layouts (1,000-sequence blocks)
    c2 = list(ref.synthesize(999, 1, preset=0, bounds=[1024], fracs=[1.0], max_length=1024)) + [37888]
    docs["c2_plan_summary"] = plan_summary(ref, c2, 8192, 1)
    # simulator predictions (pipeline.hpp) on the worked batch
    docs["simulator"] = {
        "1f1b": ref.simulate([1, 1, 2, 4], 1, 1, 4, mode=0),
        "sa_k1": ref.simulate([1, 1, 2, 4], 2, 1, 4, mode=1),
        "sa_k2": ref.simulate([1, 1, 2, 4], 2, 2, 4, mode=1),
        "sa_cs4": ref.simulate([1, 1, 2, 4], 4, 1, 4, mode=1),
    }
    with open(os.path.join(OUT, "reference_golden.json"), "w") as f:
        json.dump(docs, f, separators=(",", ":"))
    print("wrote", os.path.join(OUT, "reference_golden.json"))


def plan_summary(ref, lengths, cs, k):
    ch, sg = ref.construct_chunks(lengths, cs)
    ev, dg = ref.schedule_step(lengths, cs, k)
    return {"lengths": [int(x) for x in lengths], "chunk_size": cs, "k": k, "n_chunks": len(ch),
            "n_events": len(ev), "diag": [int(x) for x in dg.tolist()],
            "chunk_hash": int(np.bitwise_xor.reduce((ch.view(np.int64) * 1000003 + 7).ravel())),
            "segment_hash": int(np.bitwise_xor.reduce((sg.view(np.int64) * 1000003 + 11).ravel())),
            "event_hash": int(np.bitwise_xor.reduce((ev.view(np.int64) * 1000003 + 13).ravel()))}


if __name__ == "__main__":
    main()
