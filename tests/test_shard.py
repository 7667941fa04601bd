"""Sharder and record gather: LPT balance/determinism and a world-size-2
gloo run of the gather (the multi-GPU exchange step) on CPU."""

import os
import socket

import numpy as np
import pytest
import torch.multiprocessing as mp

from paper_1509_08639_b200 import shard
from paper_1509_08639_b200.synth import c3_shape


def test_lpt_covers_every_doc_once_and_is_deterministic():
    g, a, b = c3_shape(5000, seed=3)
    n, m = g + a, g + b
    s1 = shard.lpt_shards(n, m, 8)
    s2 = shard.lpt_shards(n, m, 8)
    assert all(np.array_equal(x, y) for x, y in zip(s1, s2))
    allidx = np.sort(np.concatenate(s1))
    assert np.array_equal(allidx, np.arange(n.size))
    assert all(np.all(np.diff(x) > 0) for x in s1)  # input order within a shard


def test_lpt_balances_skewed_lengths():
    g, a, b = c3_shape(20000, seed=5)
    n, m = g + a, g + b
    for world in (2, 4, 8):
        assert shard.shard_imbalance(shard.lpt_shards(n, m, world), n, m) < 1.01


def test_restore_order_is_stable_per_doc():
    r = np.zeros(5, shard.RECORD_DTYPE)
    r["doc"] = [3, 1, 3, 1, 2]
    r["i"] = [0, 0, 1, 1, 0]
    out = shard.restore_order([r[:2], r[2:]])
    assert list(zip(out["doc"], out["i"])) == [(1, 0), (1, 1), (2, 0), (3, 0), (3, 1)]


def _free_port() -> int:
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, n, m, result_path):
    import torch.distributed as dist

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    shards = shard.lpt_shards(n, m, world)
    idx = shards[rank]
    # fake per-doc records: min(n,m) // 3 records per doc, path-ordered i
    parts = []
    for d in idx:
        k = int(min(n[d], m[d]) // 3)
        r = np.zeros(k, shard.RECORD_DTYPE)
        r["doc"] = d
        r["i"] = np.arange(k)
        r["j"] = np.arange(k) * 2
        r["conf"] = 0.5 + d * 1e-6
        parts.append(r)
    recs = np.concatenate(parts) if parts else np.zeros(0, shard.RECORD_DTYPE)
    out = shard.gather_records(recs)
    if rank == 0:
        np.save(result_path, out)
    dist.barrier()
    dist.destroy_process_group()


def test_gather_records_world2_gloo(tmp_path):
    g, a, b = c3_shape(300, seed=9)
    n, m = g + a, g + b
    path = str(tmp_path / "gathered.npy")
    mp.spawn(_worker, args=(2, _free_port(), n, m, path), nprocs=2, join=True)
    got = np.load(path)
    want_doc = np.concatenate([np.full(int(min(n[d], m[d]) // 3), d) for d in range(n.size)])
    assert np.array_equal(got["doc"], want_doc)
    # path order within each doc survives the exchange
    for d in (0, 7, 123):
        sel = got[got["doc"] == d]
        assert np.array_equal(sel["i"], np.arange(sel.size))


def _mine_worker(rank, world, port, result_path):
    """A rank of the multi-GPU path with the oracle standing in for its GPU:
    generate this rank's LPT shard of one C3-shaped corpus on its own (per-
    document streams), mine it (real records), gather to rank 0 (gloo), and
    reduce per-grid-point tune counts."""
    import sys

    import torch
    import torch.distributed as dist

    from conftest import ROOT, golden

    sys.path.insert(0, os.path.join(ROOT, "oracle"))
    import oracle

    from paper_1509_08639_b200 import synth
    from paper_1509_08639_b200.classifier import load_model

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    g, a, b = c3_shape(240, seed=17)
    idx = shard.lpt_shards(g + a, g + b, world)[rank]
    sc = synth.make_corpus_native(g[idx], a[idx], b[idx], ids=idx, seed=17)
    model = load_model(golden("model5k_fwd.json"))
    hb = oracle.HostBatch(sc.packed, sc.world.packed_lexicon())
    recs, _ = oracle.mine(hb, model, 0.5, 0.2, threads=2)
    recs = recs.copy()
    recs["doc"] = idx[recs["doc"]]
    out = shard.gather_records(recs)
    pens, thrs = [0.1, 0.2, 0.8], [0.3, 0.5, 0.7]
    pred, hit = oracle.tune(hb, model, pens, thrs, sc.gold_keys(), threads=2)
    tp, th = shard.reduce_tune_counts(torch.from_numpy(pred), torch.from_numpy(hit))
    if rank == 0:
        np.save(result_path, out)
        np.save(result_path + ".tune.npy", np.stack([tp, th]))
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3])
def test_sharded_mining_and_tune_reduce_gloo(tmp_path, world):
    """world ranks mine their own shards; rank 0's gathered stream and the
    reduced tune counts equal one pass over the whole corpus."""
    import sys

    from conftest import ROOT, golden

    sys.path.insert(0, os.path.join(ROOT, "oracle"))
    import oracle

    from paper_1509_08639_b200 import synth
    from paper_1509_08639_b200.classifier import load_model

    path = str(tmp_path / "gathered.npy")
    mp.spawn(_mine_worker, args=(world, _free_port(), path), nprocs=world, join=True)
    got = np.load(path)
    g, a, b = c3_shape(240, seed=17)
    sc = synth.make_corpus_native(g, a, b, seed=17)
    model = load_model(golden("model5k_fwd.json"))
    hb = oracle.HostBatch(sc.packed, sc.world.packed_lexicon())
    want, _ = oracle.mine(hb, model, 0.5, 0.2, threads=4)
    assert got.tobytes() == want.tobytes() and got.size > 1000
    pred, hit = oracle.tune(hb, model, [0.1, 0.2, 0.8], [0.3, 0.5, 0.7], sc.gold_keys(), threads=4)
    assert np.array_equal(np.load(path + ".tune.npy"), np.stack([pred, hit]))
