"""Multi-GPU data path on one device: every rank's LPT shard
of one C3-shaped corpus is mined separately, the per-rank record buffers are
laid out as the NCCL gather delivers them on rank 0 (padded [world][stride]),
and bm_merge_shards restores global document order -- byte-identical to
mining the whole corpus at once, and to the oracle. (Only kernels that never
wait on one another run here; the collective itself is covered by the gloo
tests in test_shard.py.)"""

import numpy as np
import pytest

import paper_1509_08639_b200 as bm
from conftest import golden

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("world", [1, 2, 3, 8])
def test_sharded_mining_merges_to_the_single_gpu_stream(oracle_mod, world):
    import torch

    from paper_1509_08639_b200 import engine, shard, synth

    g, a, b = synth.c3_shape(3000, seed=31)
    sc = synth.make_corpus_native(g, a, b, seed=31)
    c = sc.packed
    model = bm.load_model(golden("model5k_fwd.json"))
    plex = sc.world.packed_lexicon()
    dc = engine.DeviceCorpus.upload(c)
    dl = engine.DeviceLexicon.upload(plex)
    whole, _ = engine.mine(dc, dl, engine.DocView.of(c), model, 0.5, 0.2)
    parts = []
    for r, idx in enumerate(shard.lpt_shards(c.n, c.m, world)):
        # each shard generated on its own, as a rank would (per-document streams)
        sub = synth.make_corpus_native(g[idx], a[idx], b[idx], ids=idx, seed=31)
        sdc = engine.DeviceCorpus.upload(sub.packed)
        sdl = engine.DeviceLexicon.upload(sub.world.packed_lexicon())
        recs, _ = engine.mine(sdc, sdl, engine.DocView.of(sub.packed), model, 0.5, 0.2)
        recs = recs.copy()
        recs["doc"] = idx[recs["doc"]]
        parts.append(recs)
    stride = max(1, max(p.size for p in parts))
    buf = np.zeros((world, stride), dtype=shard.RECORD_DTYPE)
    for r, p in enumerate(parts):
        buf[r, : p.size] = p
    dev = torch.device("cuda")
    pt = torch.from_numpy(buf.view(np.int32).reshape(world, stride, 6)).to(dev)
    lens = torch.tensor([p.size for p in parts], dtype=torch.int64, device=dev)
    merged = shard.merge_shards_device(pt, lens, c.n_docs).cpu().numpy().view(shard.RECORD_DTYPE)
    assert merged.tobytes() == whole.tobytes()
    assert merged.tobytes() == shard.restore_order(parts).tobytes()
    idx = np.arange(0, c.n_docs, 37)
    hb = oracle_mod.HostBatch(c, plex, c.src0[idx], c.n[idx], c.tgt0[idx], c.m[idx])
    want, _ = oracle_mod.mine(hb, model, 0.5, 0.2, threads=8)
    got = merged[np.isin(merged["doc"], idx)].copy()
    got["doc"] = np.searchsorted(idx, got["doc"])
    assert got.tobytes() == want.tobytes()


def test_sharded_tune_counts_sum_to_the_whole(oracle_mod):
    """C5 across ranks: bm_tune on every LPT shard, counts summed (what the
    NCCL all_reduce of shard.reduce_tune_counts adds up) == one pass."""
    from paper_1509_08639_b200 import engine, shard, synth

    sc = synth.make_corpus_native(*synth.c2_shape(600), seed=5)
    c = sc.packed
    keys = sc.gold_keys()
    model = bm.load_model(golden("model5k_fwd.json"))
    plex = sc.world.packed_lexicon()
    dc = engine.DeviceCorpus.upload(c)
    dl = engine.DeviceLexicon.upload(plex)
    pens, thrs = [0.05, 0.2, 0.4, 1.6], [0.2, 0.5, 0.8]
    whole = engine.tune_counts(dc, dl, engine.DocView.of(c), model, pens, thrs, keys)
    tot = [np.zeros_like(whole[0]), np.zeros_like(whole[1])]
    for idx in shard.lpt_shards(c.n, c.m, 3):
        p, h = engine.tune_counts(dc, dl, engine.DocView.of(c, idx), model, pens, thrs,
                                  [keys[d] for d in idx])
        tot[0] += p
        tot[1] += h
    assert np.array_equal(tot[0], whole[0]) and np.array_equal(tot[1], whole[1])
    wp, wh = oracle_mod.tune(oracle_mod.HostBatch(c, plex), model, pens, thrs, keys, threads=8)
    assert np.array_equal(whole[0], wp) and np.array_equal(whole[1], wh)
