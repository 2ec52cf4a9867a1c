"""Data-parallel partition on CPU with a world_size-2 gloo group.

Each rank takes its LPT share of the global plan's units (standalone chunks,
whole dependent groups) from the product planner (cf_plan_partition), runs
the CPU oracle on exactly those sequences with the GLOBAL normalizer, and the
gradients are summed with all_reduce — which must reproduce the single-process
full-batch result (the GPU path does the same reduction with NCCL)."""
import os
import socket

import numpy as np
import pytest
import torch.distributed as dist
import torch.multiprocessing as mp


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, q):
    import sys
    sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
    import torch

    import paper_2503_02356_b200 as cf
    from oracle.oracle import Oracle, model_cfg
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    o = Oracle()
    cfg = model_cfg(arch=1, vocab=29, d=16, heads=4, kv_heads=2, layers=2, ffn=24, seed=4)
    rng = np.random.default_rng(5)
    lengths = np.concatenate([rng.integers(2, 30, 23), [130, 75]]).astype(np.int64)
    tokens = o.gen_tokens(lengths, 29, 9)
    ids = np.arange(len(lengths), dtype=np.int64)
    norm = float((lengths - 1).sum())
    gplan = cf.Plan.build(lengths, 32, 2, ids)
    mine = gplan.partition(world, rank)
    ch, sg, ev, dg = mine.export()
    seqs = sorted({int(s) for s in sg["sequence_id"]})
    offs = np.concatenate([[0], np.cumsum(lengths)])
    sub_len = lengths[seqs]
    sub_tok = np.concatenate([tokens[offs[i]:offs[i + 1]] for i in seqs])
    loss, grads, instr = o.run_plan(cfg, sub_len, sub_tok, 32, 2, normalizer=norm, ids=np.array(seqs))
    t = torch.tensor(np.concatenate([[loss], grads]))
    dist.all_reduce(t)
    cover = torch.zeros(len(lengths), dtype=torch.int64)
    for s in seqs:
        cover[s] += 1
    dist.all_reduce(cover)
    chunk_ids = torch.zeros(len(gplan.export()[0]), dtype=torch.int64)
    for c in ch["chunk_id"]:
        chunk_ids[int(c)] += 1
    dist.all_reduce(chunk_ids)
    if rank == 0:
        fl, fg = o.backward_full(cfg, lengths, tokens)
        q.put((float(t[0]), t[1:].numpy(), fl, fg, cover.numpy(), chunk_ids.numpy(), int(instr[2]), int(instr[3])))
    dist.destroy_process_group()


@pytest.mark.timeout(300)
def test_dp_partition_allreduce_equals_full_batch():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    loss, grads, fl, fg, cover, chunk_ids, mism, viol = q.get(timeout=240)
    for p in procs:
        p.join(timeout=60)
    assert (cover == 1).all(), cover          # every sequence on exactly one rank
    assert (chunk_ids == 1).all(), chunk_ids  # every chunk exactly once, groups intact
    assert mism == 0 and viol == 0
    assert abs(loss - fl) <= 1e-12 * abs(fl)
    assert np.max(np.abs(grads - fg)) <= 1e-9 * np.max(np.abs(fg))


def test_partition_balance_and_group_integrity():
    import paper_2503_02356_b200 as cf
    lengths = np.concatenate([cf.capi.synthesize(999, b + 1, preset=0, bounds=[1024], fracs=[1.0],
                                                 max_length=1024) for b in range(8)] + [[37888] * 8]).astype(np.int64)
    g = cf.Plan.build(lengths, 8192, 1)
    gch = g.export()[0]
    for world in (2, 4, 8):
        seen = []
        for r in range(world):
            p = g.partition(world, r)
            ch, sg, ev, dg = p.export()
            assert dg["num_violations"] == 0
            seen += ch["chunk_id"].tolist()
            # dependent groups stay whole on one rank
            for gid, members in p.groups().items():
                assert set(members) <= set(ch["chunk_id"].tolist())
        assert sorted(seen) == gch["chunk_id"].tolist()
        tok = g.rank_tokens(world)
        assert tok.sum() == lengths.sum()
        assert tok.max() / tok.min() < 1.15, tok  # LPT on cost keeps ranks within 15% on tokens
