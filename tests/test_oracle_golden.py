"""Pin the CPU oracle against outputs of the reference implementation.

Every expected value here was produced by /root/reference (bimine) via
tests/golden/make_golden.py. Once these pass, the oracle is a trusted checker
for the GPU parity tests at sizes the golden files do not cover.
"""

import hashlib
import json

import numpy as np
import pytest

import paper_1509_08639_b200 as bm
from conftest import dp_cases, golden, load_docs, pairs_of, stacked, stress_lexicon
from oracle_pipeline import oracle_mine_text, oracle_tune_trace
from paper_1509_08639_b200.pack import pack_lexicon, pack_pairs


def _oracle_matrices(oracle, pairs, model, lex):
    corpus = pack_pairs(pairs)
    hb = oracle.HostBatch(corpus, pack_lexicon(lex, corpus))
    return [oracle.score_doc(hb, model, d) for d in range(len(pairs))]


@pytest.mark.parametrize("docs,smat,world", [
    ("docs40.jsonl", "S40.npz", "world500"),
    ("doc200.jsonl", None, "world5k"),
])
def test_oracle_scores_bit_exact(oracle_mod, docs, smat, world, request):
    lex, fwd, _ = request.getfixturevalue(world)
    pairs = pairs_of(load_docs(docs))
    got = _oracle_matrices(oracle_mod, pairs, fwd, lex)
    want = stacked(smat) if smat else [np.load(golden("S200.npz"))["S"]]
    for g, w in zip(got, want):
        assert g.shape == w.shape
        assert np.array_equal(g.view(np.uint64), w.view(np.uint64))


def test_oracle_scores_stress(oracle_mod):
    lex = stress_lexicon()
    model = bm.load_model(golden("model_stress.json"))
    pairs = pairs_of(load_docs("docs_stress.jsonl"))
    got = _oracle_matrices(oracle_mod, pairs, model, lex)
    for g, w in zip(got, stacked("S_stress.npz")):
        assert np.array_equal(g.view(np.uint64), w.view(np.uint64))


@pytest.mark.parametrize("name", ["dp_grid2x2.npz", "dp_s202.npz", "dp_s12_tiles.npz",
                                  "dp_quantized.npz", "dp_s31_shapes.npz"])
def test_oracle_dp_matches_reference(oracle_mod, name):
    mats = _regen(name)
    for (shape, cost, ops), S, p in zip(dp_cases(name), mats["S"], mats["p"]):
        assert S.shape == shape
        c, op, _, _ = oracle_mod.nw(S, p)
        assert c == cost or (np.isnan(c) and np.isnan(cost))
        assert np.array_equal(op, ops)


def _regen(name):
    """Rebuild the matrices of a dp_*.npz from the numpy seeds make_golden used."""
    import itertools

    S, P = [], []
    if name == "dp_grid2x2.npz":
        for vals in itertools.product([0.0, 0.25, 0.5, 0.75, 1.0], repeat=4):
            for p in (0.05, 0.25, 0.5, 1.0):
                S.append(np.array(vals).reshape(2, 2))
                P.append(p)
    elif name == "dp_s202.npz":
        r = np.random.default_rng(202)
        for _ in range(200):
            n, m = r.integers(1, 51, size=2)
            S.append(r.random((n, m)))
            P.append(float(r.uniform(0.05, 1.0)))
    elif name == "dp_s12_tiles.npz":
        r = np.random.default_rng(12)
        S = [r.random((127, 129)), r.random((128, 128)), r.random((130, 257))]
        P = [0.3] * 3
    elif name == "dp_quantized.npz":
        r = np.random.default_rng(7)
        for _ in range(60):
            n, m = r.integers(1, 40, size=2)
            S.append(r.integers(0, 5, size=(n, m)) / 4.0)
            P.append(float(r.choice([0.0, 0.125, 0.25, 0.5, 1.0])))
    elif name == "dp_s303_2000.npz":
        S = [np.random.default_rng(303).random((2000, 2000))]
        P = [0.3]
    elif name == "dp_s31_shapes.npz":
        r = np.random.default_rng(31)
        for n, m in [(300, 40), (40, 300), (129, 1), (1, 129), (256, 257), (513, 200), (700, 700)]:
            S.append(r.random((n, m)))
            P.append(0.2)
    return {"S": S, "p": P}


REGEN = _regen


@pytest.mark.parametrize("docs,tsv,bidir,t,p,world", [
    ("docs40.jsonl", "mine40_fwd.tsv", False, 0.5, 0.2, "world500"),
    ("docs40.jsonl", "mine40_bi.tsv", True, 0.5, 0.2, "world500"),
    ("docs40.jsonl", "mine40_bi_t03_p005.tsv", True, 0.3, 0.05, "world500"),
    ("doc200.jsonl", "mine200_bi.tsv", True, 0.5, 0.2, "world5k"),
    ("docs100x6.jsonl", "mine100x6_bi.tsv", True, 0.5, 0.2, "world5k"),
])
def test_oracle_mining_tsv_byte_identical(oracle_mod, docs, tsv, bidir, t, p, world, request):
    lex, fwd, bwd = request.getfixturevalue(world)
    pairs = pairs_of(load_docs(docs))
    got = oracle_mine_text(oracle_mod, pairs, fwd, bwd if bidir else None, lex, t, p)
    assert got == open(golden(tsv), encoding="utf-8").read()


def test_oracle_mining_1000_docs(oracle_mod, world500):
    lex, fwd, bwd = world500
    pairs = pairs_of(load_docs("docs1000_s77.jsonl.gz"))
    got = oracle_mine_text(oracle_mod, pairs, fwd, bwd, lex)
    want = json.load(open(golden("mine1000_bi.json")))
    assert got.count("\n") == want["lines"] == 4925
    assert hashlib.sha256(got.encode()).hexdigest() == want["sha256"]


@pytest.mark.parametrize("docs,tfile,k,grid", [
    ("docs40.jsonl", "tune10.json", 10, None),
    ("docs10_noisy.jsonl", "tune_noisy.json", 10, None),
    ("docs10_noisy.jsonl", "tune_noisy_small.json", 3, ([0.3, 0.6], [0.1, 0.4])),
])
def test_oracle_tune_trace(oracle_mod, world500, docs, tfile, k, grid):
    lex, fwd, _ = world500
    raw = load_docs(docs)[:k]
    dev = bm.GoldSet(docs=pairs_of(raw), gold=[{(i, j) for i, j in d["gold"]} for d in raw])
    t_grid, p_grid = grid if grid else (list(bm.tuner.DEFAULT_THRESHOLDS), list(bm.tuner.DEFAULT_PENALTIES))
    got = oracle_tune_trace(oracle_mod, fwd, lex, dev, t_grid, p_grid)
    want = json.load(open(golden(tfile)))["trace"]
    assert len(got) == len(want)
    for g, w in zip(got, want):
        assert g == (w["threshold"], w["penalty"], w["precision"], w["recall"], w["f1"])
