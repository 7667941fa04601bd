"""GPU parity at the BASELINE configs' full sizes.

* C4: the 8192 x 8192 pair, DP-only on the reference's random matrix (seed
  303, test_acceptance.py:134-142 shape) and as a full document (scored, then
  aligned and extracted), with MAX_CELLS raised as the reference's own tests
  do (test_aligner.py:315).
* C3: skewed documents up to 2000 x 2000 sentences -- the banded tier's fat
  tail (n, m = 2000, 1000 x 2000, 2000 x 10, ...) next to a C3-distributed
  sample -- against the oracle, records and costs bit for bit.
"""

import os

import numpy as np
import pytest

import paper_1509_08639_b200 as bm
from conftest import golden, moves_from_ops

pytestmark = pytest.mark.gpu

C4 = 8192


def bits(a):
    return np.ascontiguousarray(a, dtype=np.float64).view(np.uint64)


def test_c4_dp_8192_random_vs_oracle(oracle_mod, monkeypatch):
    """aligner.py:116-134 + :176-206 on the 67M-cell random matrix."""
    monkeypatch.setattr(bm.aligner, "MAX_CELLS", C4 * C4)
    S = np.random.default_rng(303).random((C4, C4))
    for p in (0.3, 0.05):
        got = bm.nw_align(bm.SimilarityMatrix(S), p)
        c, ops, _, _ = oracle_mod.nw(S, p)
        assert got.total_cost == c
        assert got.moves == moves_from_ops(ops)


def test_c4_full_document_vs_oracle(oracle_mod, monkeypatch):
    """One 8192 x 8192 synthetic document: S (aligner.py:313-339) bit-exact,
    then the mined records and path cost (miner.py:84-128)."""
    from paper_1509_08639_b200 import engine, synth

    monkeypatch.setattr(bm.aligner, "MAX_CELLS", C4 * C4)
    sc = synth.make_corpus([4915], [C4 - 4915], [C4 - 4915], seed=404)
    c = sc.packed
    assert int(c.n[0]) == C4 and int(c.m[0]) == C4
    model = bm.load_model(golden("model5k_fwd.json"))
    plex = sc.world.packed_lexicon()
    dc = engine.DeviceCorpus.upload(c)
    dl = engine.DeviceLexicon.upload(plex)
    view = engine.DocView.of(c)
    S, s_off, pitch, _, _ = engine.score(dc, dl, view, model)
    got_S = engine.matrices_from_buffer(S, s_off, pitch, view.n, view.m)[0]
    del S
    hb = oracle_mod.HostBatch(c, plex)
    want_S = oracle_mod.score_doc(hb, model, 0)
    assert np.array_equal(bits(got_S), bits(want_S))
    for t, p in ((0.5, 0.2), (0.3, 0.05)):
        recs, cost = engine.mine(dc, dl, view, model, t, p)
        want, wcost = oracle_mod.mine(hb, model, t, p, threads=1)
        assert np.array_equal(bits(cost), bits(wcost))
        assert recs.tobytes() == want.tobytes()
    # the DP on the scored matrix through the API equals the fused mining path
    path = bm.nw_align(bm.SimilarityMatrix(got_S), 0.2)
    c2, ops, _, _ = oracle_mod.nw(want_S, 0.2)
    assert path.total_cost == c2 and path.moves == moves_from_ops(ops)


def _c3_tail_corpus(seed: int):
    from paper_1509_08639_b200 import synth

    tail = [(2000, 2000), (1000, 2000), (2000, 1000), (2000, 10), (10, 2000), (1999, 1998),
            (257, 300), (700, 1500), (256, 2000), (129, 130), (1500, 257), (384, 384)]
    g, a, b = synth.c3_shape(400, seed=seed)
    n = np.r_[[t[0] for t in tail], g + a]
    m = np.r_[[t[1] for t in tail], g + b]
    gold = (0.6 * np.minimum(n, m)).astype(np.int64)
    return synth.make_corpus(gold, n - gold, m - gold, seed=seed)


@pytest.mark.parametrize("seed", [2026, 7])
def test_c3_tail_documents_vs_oracle(oracle_mod, seed):
    from paper_1509_08639_b200 import engine

    sc = _c3_tail_corpus(seed)
    c = sc.packed
    assert int(c.n.max()) == 2000 and int(c.m.max()) == 2000
    model = bm.load_model(golden("model5k_fwd.json"))
    plex = sc.world.packed_lexicon()
    dc = engine.DeviceCorpus.upload(c)
    dl = engine.DeviceLexicon.upload(plex)
    view = engine.DocView.of(c)
    hb = oracle_mod.HostBatch(c, plex)
    for t, p in ((0.5, 0.2), (0.4, 0.8)):
        recs, cost = engine.mine(dc, dl, view, model, t, p)
        want, wcost = oracle_mod.mine(hb, model, t, p, threads=os.cpu_count() or 8)
        assert np.array_equal(bits(cost), bits(wcost))
        assert recs.tobytes() == want.tobytes()


def test_c3_tail_tune_vs_oracle(oracle_mod):
    """K5 over the same fat-tailed documents: pred/hit counts per grid point."""
    from paper_1509_08639_b200 import engine

    sc = _c3_tail_corpus(11)
    c = sc.packed
    model = bm.load_model(golden("model5k_fwd.json"))
    plex = sc.world.packed_lexicon()
    keys = [np.asarray(gd[:, 0] * int(c.m[d]) + gd[:, 1], np.int64) for d, gd in enumerate(sc.gold)]
    pens, thrs = [0.05, 0.2, 0.4, 1.6, 0.1], [0.3, 0.5, 0.7]
    p, h = engine.tune_counts(engine.DeviceCorpus.upload(c), engine.DeviceLexicon.upload(plex),
                              engine.DocView.of(c), model, pens, thrs, keys)
    wp, wh = oracle_mod.tune(oracle_mod.HostBatch(c, plex), model, pens, thrs, keys,
                             threads=os.cpu_count() or 8)
    assert np.array_equal(p, wp) and np.array_equal(h, wh)


@pytest.mark.parametrize("seed", [2026, 7])
def test_band_parallel_extraction_vs_oracle(seed):
    """The band-parallel extraction (exit maps per band, one warp per band,
    band-ordered gather) on every tail document with n > 512 and n + m >= 600
    (BM_PAR_WALK_MIN=600 in a child process), next to serially extracted
    documents of the same plan: records and costs equal the oracle's."""
    import subprocess
    import sys

    env = dict(os.environ, BM_PAR_WALK_MIN="600")
    child = os.path.join(os.path.dirname(os.path.abspath(__file__)), "par_walk_child.py")
    r = subprocess.run([sys.executable, child, str(seed)], env=env, capture_output=True, text=True,
                       timeout=600)
    assert r.returncode == 0, r.stdout[-2000:] + r.stderr[-4000:]
    assert "records equal" in r.stdout


@pytest.mark.parametrize("env", [
    {"BM_BAND_FUSED": "1", "BM_BAND_MIN_ITEMS": "1"},
    {"BM_BAND_FUSED": "1", "BM_BAND_MIN_ITEMS": "1", "BM_PAR_WALK_MIN": "600"},
    {"BM_DP_OVERLAP": "1"},
])
def test_fused_band_tier_vs_oracle(env):
    """The opt-in routes in child processes: the fused banded tier
    (mine_band_kernel: scoring warps feeding the DP warp through a
    shared-memory ring, no similarity matrix; extraction re-scores the path
    cells) with serial and band-parallel extraction, and the DP overlapped with
    the scoring kernel (per-band readiness counters); four penalties including
    inf: records and costs equal the oracle's."""
    import subprocess
    import sys

    child = os.path.join(os.path.dirname(os.path.abspath(__file__)), "par_walk_child.py")
    r = subprocess.run([sys.executable, child, "2026"], env=dict(os.environ, **env),
                       capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stdout[-2000:] + r.stderr[-4000:]
    assert "records equal" in r.stdout
