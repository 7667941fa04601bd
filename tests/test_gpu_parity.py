"""GPU parity: the sm_100a path against the reference's golden outputs and the
(pinned) CPU oracle. Bit-exact for every score, cost, path and record."""

import hashlib
import io
import json
import math

import numpy as np
import pytest

import paper_1509_08639_b200 as bm
from conftest import dp_cases, golden, load_docs, moves_from_ops, pairs_of, stacked, stress_lexicon
from oracle_pipeline import oracle_mine_text
from test_oracle_golden import REGEN

pytestmark = pytest.mark.gpu


def bits(a):
    return np.ascontiguousarray(a, dtype=np.float64).view(np.uint64)


# ---------------------------------------------------------------- K1 scoring
def test_scores_docs40_bit_exact(world500):
    lex, fwd, _ = world500
    got = bm.build_similarity_matrices(pairs_of(load_docs("docs40.jsonl")), fwd, lex)
    for g, w in zip(got, stacked("S40.npz")):
        assert np.array_equal(bits(g.cells), bits(w))


def test_scores_200x200_bit_exact(world5k):
    lex, fwd, _ = world5k
    got = bm.build_similarity_matrix(pairs_of(load_docs("doc200.jsonl"))[0], fwd, lex)
    assert np.array_equal(bits(got.cells), bits(np.load(golden("S200.npz"))["S"]))


def test_scores_stress_bit_exact():
    lex = stress_lexicon()
    model = bm.load_model(golden("model_stress.json"))
    got = bm.build_similarity_matrices(pairs_of(load_docs("docs_stress.jsonl")), model, lex)
    for g, w in zip(got, stacked("S_stress.npz")):
        assert np.array_equal(bits(g.cells), bits(w))


def test_confidence_exp_sweep(oracle_mod):
    """bm_confidence over 200k margins == libm-based oracle (glibc exp port)."""
    rng = np.random.default_rng(1)
    z = np.concatenate([rng.uniform(-40, 40, 150000), rng.uniform(-800, 800, 50000),
                        [0.0, -0.0, 1e-300, -1e-300, 700.0, -745.0, -1100.0]])
    feats = np.zeros((z.size, 7))
    feats[:, 0] = 1.0
    model = bm.ClassifierModel("pairwise-v1", [1.0] + [0.0] * 6, 0.0, ("a", "b"), 0.5, 0.2)
    from paper_1509_08639_b200 import engine

    out = np.empty(z.size)
    for k0 in range(0, z.size, 50000):
        f = feats[k0 : k0 + 50000].copy()
        f[:, 0] = z[k0 : k0 + 50000]
        out[k0 : k0 + 50000] = engine.confidences(f, model)
    w = np.array([1.0] + [0.0] * 6)
    import ctypes

    want = np.array([oracle_mod.lib().oracle_confidence(w.ctypes.data, 0.0,
                     np.array([x, 0, 0, 0, 0, 0, 0.0]).ctypes.data) for x in z])
    assert np.array_equal(bits(out), bits(want))


def test_single_cell_confidence_known_answer():
    # test_miner.py:79-93: all-zero weights, bias 2 -> sigmoid(2)
    model = bm.ClassifierModel("pairwise-v1", [0.0] * 7, 2.0, ("xx", "yy"), 0.5, 0.2)
    f = bm.FeatureVector(values=[0.3, 0.9, 0.1, 1.0, 0.5, 0.7, 1.0])
    assert bm.confidence(model, f) == 1.0 / (1.0 + math.exp(-2.0))
    zero = bm.ClassifierModel("pairwise-v1", [0.0] * 7, 0.0, ("xx", "yy"), 0.5, 0.2)
    assert bm.confidence(zero, f) == 0.5


def test_features_and_coverage_vs_oracle(oracle_mod):
    lex = stress_lexicon()
    pairs = pairs_of(load_docs("docs_stress.jsonl"))
    sents_s = [s for p in pairs for s in p.source.sentences]
    sents_t = [s for p in pairs for s in p.target.sentences]
    rng = np.random.default_rng(3)
    items = [(sents_s[rng.integers(len(sents_s))], sents_t[rng.integers(len(sents_t))],
              float(rng.random()), float(rng.random())) for _ in range(64)]
    got = bm.classifier._features_batch(items, lex)
    from paper_1509_08639_b200.pack import Packer, pack_lexicon

    pk = Packer()
    idx = [pk.add_sentence_pair(a, b) for a, b, _, _ in items]
    corpus = pk.finish()
    hb = oracle_mod.HostBatch(corpus, pack_lexicon(lex, corpus))
    for k, ((a, b), (_, _, ps, pt)) in enumerate(zip(idx, items)):
        want = oracle_mod.features(hb, a, b, ps, pt)
        assert np.array_equal(bits(got[k]), bits(want))
    # the lexicon.coverage API primitive (lexicon.py:88-105 known answers)
    simple = bm.Lexicon(("xx", "yy"), {"hund": [("dog", 0.9)], "katze": [("cat", 0.8)]})
    assert bm.coverage(simple, ["hund", "katze"], ["dog", "fish"]) == 0.5
    assert bm.coverage(simple, ["Hund"], ["DOG"]) == 1.0
    assert bm.coverage(simple, ["42", "."], ["dog"]) == 0.0


# ---------------------------------------------------------------- K2/K3/K4a DP
@pytest.mark.parametrize("name", ["dp_grid2x2.npz", "dp_s202.npz", "dp_s12_tiles.npz",
                                  "dp_quantized.npz", "dp_s31_shapes.npz", "dp_s303_2000.npz"])
def test_dp_matches_reference(name):
    mats = REGEN(name)
    cases = dp_cases(name)
    by_p: dict[float, list[int]] = {}
    for k, p in enumerate(mats["p"]):
        by_p.setdefault(p, []).append(k)
    for p, ks in by_p.items():
        paths = bm.aligner.align_many([bm.SimilarityMatrix(mats["S"][k]) for k in ks], p)
        for k, path in zip(ks, paths):
            shape, cost, ops = cases[k]
            assert path.total_cost == cost
            assert path.moves == moves_from_ops(ops)


def test_dp_known_answers():
    # test_aligner.py:150-177
    p = bm.nw_align(bm.SimilarityMatrix(np.array([[1.0, 0.0], [0.0, 1.0]])), 0.5)
    assert p.total_cost == 0.0 and [m.op for m in p.moves] == ["D", "D"]
    p = bm.nw_align(bm.SimilarityMatrix(np.array([[0.9]])), 0.5)
    assert p.moves == [bm.Move("D", 0, 0)] and abs(p.total_cost - 0.1) < 1e-12
    p = bm.nw_align(bm.SimilarityMatrix(np.zeros((2, 2))), 0.1)
    assert [m.op for m in p.moves] == ["GT", "GT", "GS", "GS"]
    p = bm.nw_align(bm.SimilarityMatrix(np.array([[1.0, 1.0]])), 0.2)
    assert [m.op for m in p.moves].count("GT") == 1
    S = bm.SimilarityMatrix(np.array([[0.9, 0.0], [0.0, 0.8]]))
    assert bm.format_path(bm.nw_align(S, 0.5), S) == ["D 0 0 0.100000", "D 1 1 0.200000",
                                                       "TOTAL 0.300000"]


def test_dp_penalty_edges(oracle_mod):
    rng = np.random.default_rng(9)
    for p in (0.0, float("inf"), 1e300, 5e-324):
        for shape in ((1, 1), (3, 7), (200, 150)):
            S = rng.random(shape)
            got = bm.nw_align(bm.SimilarityMatrix(S), p)
            c, ops, _, _ = oracle_mod.nw(S, p)
            assert (got.total_cost == c) or (math.isnan(c) and math.isnan(got.total_cost))
            assert got.moves == moves_from_ops(ops)
    with pytest.raises(ValueError, match="penalty"):
        bm.nw_align(bm.SimilarityMatrix(np.eye(2)), -0.1)
    with pytest.raises(ValueError, match="penalty"):
        bm.nw_align(bm.SimilarityMatrix(np.eye(2)), float("nan"))


def test_dp_long_pair_vs_oracle(oracle_mod):
    """A 4096 x 3000 DP (multi-band, inter-warp boundary handoff)."""
    S = np.random.default_rng(4).random((4096, 3000))
    got = bm.nw_align(bm.SimilarityMatrix(S), 0.25)
    c, ops, _, _ = oracle_mod.nw(S, 0.25)
    assert got.total_cost == c
    assert got.moves == moves_from_ops(ops)


def test_extract_pairs_api(world500):
    lex, fwd, _ = world500
    pair = pairs_of(load_docs("docs40.jsonl"))[0]
    S = bm.build_similarity_matrix(pair, fwd, lex)
    path = bm.nw_align(S, 0.2)
    got = bm.extract_pairs(path, S, pair, bm.MiningParams(0.5, 0.2))
    want = [(mv.i, mv.j) for mv in path.moves if mv.op == "D" and S.cells[mv.i, mv.j] >= 0.5]
    assert [(r.src_index, r.tgt_index) for r in got] == want
    assert all(r.confidence == S.cells[r.src_index, r.tgt_index] for r in got)


# ---------------------------------------------------------------- mining
def _mine_text(pairs, fwd, bwd, lex, t=0.5, p=0.2):
    sink = io.StringIO()
    rep = bm.mine_corpus(iter(pairs), fwd, bwd, lex, bm.MinerConfig(bm.MiningParams(t, p)), sink)
    rep.wall_clock_seconds = 0.0
    return sink.getvalue(), bm.report_to_json(rep)


@pytest.mark.parametrize("docs,tsv,bidir,t,p,world", [
    ("docs40.jsonl", "mine40_fwd.tsv", False, 0.5, 0.2, "world500"),
    ("docs40.jsonl", "mine40_bi.tsv", True, 0.5, 0.2, "world500"),
    ("docs40.jsonl", "mine40_bi_t03_p005.tsv", True, 0.3, 0.05, "world500"),
    ("doc200.jsonl", "mine200_fwd.tsv", False, 0.5, 0.2, "world5k"),
    ("doc200.jsonl", "mine200_bi.tsv", True, 0.5, 0.2, "world5k"),
    ("docs100x6.jsonl", "mine100x6_bi.tsv", True, 0.5, 0.2, "world5k"),
])
def test_mine_corpus_tsv_byte_identical(docs, tsv, bidir, t, p, world, request):
    lex, fwd, bwd = request.getfixturevalue(world)
    text, rep = _mine_text(pairs_of(load_docs(docs)), fwd, bwd if bidir else None, lex, t, p)
    assert text == open(golden(tsv), encoding="utf-8").read()
    if tsv in ("mine40_fwd.tsv", "mine40_bi.tsv"):
        assert rep == open(golden(tsv.replace(".tsv", ".report.json"))).read()


@pytest.mark.parametrize("docs,tsv,bidir,t,p,world", [
    ("docs40.jsonl", "mine40_fwd.tsv", False, 0.5, 0.2, "world500"),
    ("docs40.jsonl", "mine40_bi.tsv", True, 0.5, 0.2, "world500"),
    ("docs40.jsonl", "mine40_bi_t03_p005.tsv", True, 0.3, 0.05, "world500"),
    ("doc200.jsonl", "mine200_fwd.tsv", False, 0.5, 0.2, "world5k"),
    ("doc200.jsonl", "mine200_bi.tsv", True, 0.5, 0.2, "world5k"),
    ("docs100x6.jsonl", "mine100x6_bi.tsv", True, 0.5, 0.2, "world5k"),
])
def test_mine_corpus_file_native_path_byte_identical(docs, tsv, bidir, t, p, world, request):
    """Native JSONL reader + lexicon lowering + merge/TSV emission (ingest.py):
    the reference's TSV bytes and report."""
    from paper_1509_08639_b200.ingest import NativeCorpus

    lex, fwd, bwd = request.getfixturevalue(world)
    path = golden(docs)
    assert NativeCorpus.load(path) is not None  # ASCII fixtures take the native path
    sink = io.StringIO()
    rep = bm.mine_corpus_file(path, fwd, bwd if bidir else None, lex,
                              bm.MinerConfig(bm.MiningParams(t, p)), sink)
    rep.wall_clock_seconds = 0.0
    assert sink.getvalue() == open(golden(tsv), encoding="utf-8").read()
    if tsv in ("mine40_fwd.tsv", "mine40_bi.tsv"):
        assert bm.report_to_json(rep) == open(golden(tsv.replace(".tsv", ".report.json"))).read()


@pytest.mark.parametrize("workers", [1, 3])
@pytest.mark.parametrize("entry", ["mine_corpus", "mine_corpus_file"])
def test_mine_corpus_malformed_line_after_good_docs(world500, tmp_path, workers, entry):
    """A loader error after 5 good documents (tests/golden/make_golden_r02.py):
    workers=1 writes those 5 documents first, workers>1 writes nothing, and
    the loader's DataError propagates either way -- the reference's bytes."""
    lex, fwd, bwd = world500
    lines = open(golden("docs40.jsonl"), encoding="utf-8").read().splitlines(True)
    path = str(tmp_path / "bad.jsonl")
    with open(path, "w", encoding="utf-8") as fh:
        fh.writelines(lines[:5])
        fh.write("{not json\n")
        fh.writelines(lines[5:])
    want = json.load(open(golden("mine40_badline.json")))[f"workers{workers}"]
    sink = io.StringIO()
    cfg = bm.MinerConfig(bm.MiningParams(0.5, 0.2), workers=workers)
    with pytest.raises(bm.DataError) as exc:
        if entry == "mine_corpus":
            bm.mine_corpus(bm.load_document_pairs(path), fwd, bwd, lex, cfg, sink)
        else:
            bm.mine_corpus_file(path, fwd, bwd, lex, cfg, sink)
    assert str(exc.value).replace(path, "<path>") == want["error"]
    assert sink.getvalue() == want["tsv"]


def test_mine_corpus_file_1000_docs_sha256(world500, tmp_path):
    import gzip

    lex, fwd, bwd = world500
    p = str(tmp_path / "docs1000.jsonl")
    with gzip.open(golden("docs1000_s77.jsonl.gz"), "rb") as fi, open(p, "wb") as fo:
        fo.write(fi.read())
    sink = io.StringIO()
    bm.mine_corpus_file(p, fwd, bwd, lex, bm.MinerConfig(bm.MiningParams(0.5, 0.2)), sink)
    want = json.load(open(golden("mine1000_bi.json")))
    text = sink.getvalue()
    assert text.count("\n") == want["lines"]
    assert hashlib.sha256(text.encode()).hexdigest() == want["sha256"]


def test_mine_corpus_file_unicode_native_path(tmp_path):
    """Non-ASCII corpora take the native path too: docs40 and its lexicon with
    every 'a'/'A' spelled 'ą'/'Ą' (two UTF-8 bytes; no abbreviation contains
    'a', so segmentation is unchanged) mine to the golden TSV spelled the same
    way, through raw UTF-8 lines and \\u-escaped lines alike."""
    from paper_1509_08639_b200.ingest import NativeCorpus

    tr = str.maketrans({"a": "\u0105", "A": "\u0104"})
    lp = tmp_path / "lex.tsv"
    lp.write_text(open(golden("lex500.tsv"), encoding="utf-8").read().translate(tr),
                  encoding="utf-8")
    lex = bm.load_lexicon(str(lp), "xx", "yy")
    fwd = bm.load_model(golden("model500_fwd.json"))
    bwd = bm.load_model(golden("model500_bwd.json"))
    p = str(tmp_path / "docs.jsonl")
    with open(p, "w", encoding="utf-8") as fh:
        for q, d in enumerate(load_docs("docs40.jsonl")):
            for side in ("src", "tgt"):
                d[side] = (d[side].translate(tr) if isinstance(d[side], str)
                           else [s.translate(tr) for s in d[side]])
            fh.write(json.dumps(d, ensure_ascii=bool(q % 2)) + "\n")
    assert NativeCorpus.load(p) is not None
    sink = io.StringIO()
    bm.mine_corpus_file(p, fwd, bwd, lex, bm.MinerConfig(bm.MiningParams(0.5, 0.2)), sink)
    want = []
    for line in open(golden("mine40_bi.tsv"), encoding="utf-8").read().splitlines(True):
        cols = line.split("\t")
        want.append("\t".join([cols[0].translate(tr), cols[1].translate(tr)] + cols[2:]))
    assert "\u0105" in sink.getvalue()
    assert sink.getvalue() == "".join(want)


def test_mine_corpus_file_falls_back_outside_the_subset(world500, tmp_path):
    """Text NFC would change takes the Python reader: same output as mine_corpus."""
    lex, fwd, bwd = world500
    docs = load_docs("docs40.jsonl")[:5]
    docs[1]["src"][0] = docs[1]["src"][0] + " cafe\u0301"
    p = str(tmp_path / "mixed.jsonl")
    with open(p, "w", encoding="utf-8") as fh:
        for d in docs:
            fh.write(json.dumps(d, ensure_ascii=False) + "\n")
    cfg = bm.MinerConfig(bm.MiningParams(0.5, 0.2))
    a, b = io.StringIO(), io.StringIO()
    bm.mine_corpus_file(p, fwd, bwd, lex, cfg, a)
    bm.mine_corpus(bm.load_document_pairs(p), fwd, bwd, lex, cfg, b)
    assert a.getvalue() == b.getvalue() and a.getvalue()


def test_mine_corpus_1000_docs_sha256(world500):
    lex, fwd, bwd = world500
    text, _ = _mine_text(pairs_of(load_docs("docs1000_s77.jsonl.gz")), fwd, bwd, lex)
    want = json.load(open(golden("mine1000_bi.json")))
    assert text.count("\n") == want["lines"]
    assert hashlib.sha256(text.encode()).hexdigest() == want["sha256"]


def test_mine_document_orientation_and_errors(world500):
    lex, fwd, bwd = world500
    pair = pairs_of(load_docs("docs40.jsonl"))[3]
    cfg = bm.MinerConfig(bm.MiningParams(0.5, 0.2))
    got = bm.mine_document(pair, bwd, lex.reversed(), cfg)
    assert got and all(r.direction == "backward" for r in got)
    for engine_name in bm.ENGINES:
        a = bm.mine_document(pair, fwd, lex, bm.MinerConfig(bm.MiningParams(0.5, 0.2), engine=engine_name))
        assert a == bm.mine_document(pair, fwd, lex, cfg)
    with pytest.raises(bm.DataError, match="lexicon direction"):
        bm.mine_document(pair, fwd, lex.reversed(), cfg)


def test_mine_corpus_skips_over_cap(world500, monkeypatch):
    lex, fwd, _ = world500
    pairs = pairs_of(load_docs("docs40.jsonl"))[:5]
    monkeypatch.setattr("paper_1509_08639_b200.aligner.MAX_CELLS", 16)
    rep = bm.mine_corpus(iter(pairs), fwd, None, lex, bm.MinerConfig(bm.MiningParams(0.5, 0.2)),
                         io.StringIO())
    assert rep.docs_skipped == 5 and rep.docs_processed == 0


def _synth_mixed(seed):
    from paper_1509_08639_b200 import synth

    r = np.random.default_rng(seed)
    D = 96
    n = r.integers(1, 420, D)
    m = r.integers(1, 420, D)
    n[:6] = [1, 1, 300, 257, 40, 700]
    m[:6] = [1, 300, 1, 100, 700, 40]
    g = np.minimum(n, m) // 2
    return synth.make_corpus(g, n - g, m - g, vocab=2000, seed=seed)


@pytest.mark.parametrize("seed", [5, 6])
def test_mine_mixed_sizes_vs_oracle(oracle_mod, seed):
    """Docs routed to both tiers (fused warp-per-doc and banded) == oracle."""
    from paper_1509_08639_b200 import engine

    sc = _synth_mixed(seed)
    model = bm.load_model(golden("model5k_fwd.json"))
    plex = sc.world.packed_lexicon()
    dc = engine.DeviceCorpus.upload(sc.packed)
    dl = engine.DeviceLexicon.upload(plex)
    view = engine.DocView.of(sc.packed)
    # 0 and inf: the DP's edge penalties (inf keeps the literal compare order)
    for t, p in ((0.5, 0.2), (0.2, 0.05), (0.5, 0.0), (0.4, float("inf"))):
        recs, cost = engine.mine(dc, dl, view, model, t, p)
        hb = oracle_mod.HostBatch(sc.packed, plex)
        want, wcost = oracle_mod.mine(hb, model, t, p, threads=8)
        assert np.array_equal(bits(cost), bits(wcost))
        assert recs.shape == want.shape
        for f in ("doc", "i", "j"):
            assert np.array_equal(recs[f], want[f])
        assert np.array_equal(bits(recs["conf"]), bits(want["conf"]))


def test_mine_long_sentences_general_path(oracle_mod):
    """A sentence with > 255 alpha tokens forces the 32-bit-hit banded path."""
    long_src = " ".join(["waaa"] * 300 + ["wbbb"] * 10) + "."
    long_tgt = " ".join(["vaaa"] * 280) + " 1999."
    doc = {"id": "long", "src_lang": "xx", "tgt_lang": "yy",
           "src": ["waaa wbbb.", long_src, "wccc 1999."], "tgt": [long_tgt, "vaaa vbbb.", "vccc."]}
    lex = bm.Lexicon(("xx", "yy"), {"waaa": [("vaaa", 0.9)], "wbbb": [("vbbb", 0.9)],
                                     "wccc": [("vccc", 0.9)]})
    model = bm.load_model(golden("model5k_fwd.json"))
    pairs = pairs_of([doc])
    cfg = bm.MinerConfig(bm.MiningParams(0.1, 0.3))
    got = bm.mine_document(pairs[0], model, lex, cfg)
    from oracle_pipeline import oracle_records

    recs, _ = oracle_records(oracle_mod, pairs, model, lex, [False], 0.1, 0.3)
    assert [(r.src_index, r.tgt_index, r.confidence) for r in got] == \
        [(int(a), int(b), float(c)) for a, b, c in zip(recs["i"], recs["j"], recs["conf"])]


def _big_token_docs():
    """tests/golden/make_golden_r02.py big_token_docs(): a document whose first
    sentences hold 70,003 / 66,002 tokens (multiplicities and hit counts past
    16 bits) between two docs40 documents."""
    docs = load_docs("docs40.jsonl")[:3]
    big = dict(docs[1], id="big")
    big["src"] = ["waaa " * 70000 + "wadf walb."] + docs[1]["src"][1:]
    big["tgt"] = ["vaaa " * 66000 + "vadf vafr."] + docs[1]["tgt"][1:]
    return [docs[0], big, docs[2]]


def test_sentences_over_65535_tokens_are_mined(world500, tmp_path):
    """Sentences longer than 65,535 tokens are mined like any other (32-bit
    counts on the per-tile scoring path): the reference's TSV bytes and report,
    through both the Python and the native JSONL paths."""
    lex, fwd, bwd = world500
    want = json.load(open(golden("mine_big_tokens.json")))
    docs = _big_token_docs()
    got, rep = _mine_text(pairs_of(docs), fwd, bwd, lex)
    assert hashlib.sha256(got.encode()).hexdigest() == want["sha256"]
    assert rep == want["report"]
    assert [ln for ln in got.splitlines(True) if len(ln) < 400] == want["short_lines"]
    p = str(tmp_path / "big.jsonl")
    with open(p, "w") as fh:
        for d in docs:
            fh.write(json.dumps(d) + "\n")
    sink = io.StringIO()
    rep2 = bm.mine_corpus_file(p, fwd, bwd, lex, bm.MinerConfig(bm.MiningParams(0.5, 0.2)), sink)
    assert hashlib.sha256(sink.getvalue().encode()).hexdigest() == want["sha256"]
    assert rep2.docs_skipped == 0 and rep2.pairs_emitted == want["lines"]


def test_big_token_scores_and_tune_vs_oracle(world500, oracle_mod):
    """The same document's similarity matrix (bm_score) and a tune sweep over it
    (bm_tune with token_bound > 65535) against the oracle."""
    from oracle_pipeline import oracle_records  # noqa: F401
    from paper_1509_08639_b200 import engine
    from paper_1509_08639_b200.pack import pack_lexicon, pack_pairs

    lex, fwd, _ = world500
    pairs = pairs_of(_big_token_docs())
    S = bm.build_similarity_matrix(pairs[1], fwd, lex).cells
    corpus = pack_pairs(pairs)
    hb = oracle_mod.HostBatch(corpus, pack_lexicon(lex, corpus))
    want = oracle_mod.score_doc(hb, fwd, 1)
    assert np.array_equal(S.view(np.uint64), want.view(np.uint64))
    gold = [np.asarray([0, 1 * int(corpus.m[d]) + 1], np.int64) for d in range(3)]
    dc = engine.DeviceCorpus.upload(corpus)
    dl = engine.DeviceLexicon.upload(pack_lexicon(lex, corpus))
    assert dc.max_tok > 65535
    p, h = engine.tune_counts(dc, dl, engine.DocView.of(corpus), fwd, [0.1, 0.2, 0.4],
                              [0.3, 0.5, 0.9], gold)
    wp, wh = oracle_mod.tune(hb, fwd, [0.1, 0.2, 0.4], [0.3, 0.5, 0.9], gold)
    assert np.array_equal(p, wp) and np.array_equal(h, wh)


def test_synth_text_round_trip_same_records():
    """Packed-by-generator and packed-from-text corpora mine identically."""
    from paper_1509_08639_b200 import engine, synth
    from paper_1509_08639_b200.pack import pack_lexicon, pack_pairs

    sc = synth.make_corpus(*synth.c2_shape(40), seed=8)
    model = bm.load_model(golden("model5k_fwd.json"))
    a, _ = engine.mine(engine.DeviceCorpus.upload(sc.packed),
                       engine.DeviceLexicon.upload(sc.world.packed_lexicon()),
                       engine.DocView.of(sc.packed), model, 0.5, 0.2)
    pairs = sc.doc_pairs(range(40))
    pc = pack_pairs(pairs)
    b, _ = engine.mine(engine.DeviceCorpus.upload(pc),
                       engine.DeviceLexicon.upload(pack_lexicon(sc.world.lexicon(), pc)),
                       engine.DocView.of(pc), model, 0.5, 0.2)
    assert a.tobytes() == b.tobytes()


@pytest.mark.parametrize("wire,pin", [(False, False), ("wire", False), ("wire", True), (False, True),
                                      ("packed", False), ("packed", True)])
def test_mine_host_entry_point_matches_device_path(oracle_mod, wire, pin):
    """bm_mine_host / _wire / _packed (host buffers in, records out) == oracle,
    from pageable and from page-locked host buffers."""
    from paper_1509_08639_b200 import hostapi, synth

    sc = synth.make_corpus(*synth.c2_shape(3000), seed=11)  # several streamed chunks
    model = bm.load_model(golden("model5k_fwd.json"))
    plex = sc.world.packed_lexicon()
    assert hostapi.wire_ok(sc.packed, plex) and hostapi.packed_ok(sc.packed, plex)
    recs, cost = hostapi.mine_host(sc.packed, plex, model, 0.5, 0.2, wire=wire, pin=pin)
    want, wcost = oracle_mod.mine(oracle_mod.HostBatch(sc.packed, plex), model, 0.5, 0.2, threads=16)
    assert recs.tobytes() == want.tobytes()
    assert np.array_equal(bits(cost), bits(wcost))


def test_mine_host_formats_on_a_skewed_corpus():
    """Skewed document sizes put chunk boundaries at arbitrary sentence indices
    (not multiples of the packed format's 32-sentence blocks) and route some
    documents to the banded tier: every host format == the device path."""
    from paper_1509_08639_b200 import engine, hostapi, synth

    g, a, b = synth.c3_shape(1500, seed=5)
    sc = synth.make_corpus(g, a, b, seed=5)
    c, plex = sc.packed, sc.world.packed_lexicon()
    model = bm.load_model(golden("model5k_fwd.json"))
    assert int((c.n.astype(np.int64) * c.m).sum()) > 20 << 20  # several chunks
    want, wcost = engine.mine(engine.DeviceCorpus.upload(c), engine.DeviceLexicon.upload(plex),
                              engine.DocView.of(c), model, 0.5, 0.2)
    for fmt in ("packed", "wire", False):
        recs, cost = hostapi.mine_host(c, plex, model, 0.5, 0.2, wire=fmt, pin=True)
        assert recs.tobytes() == want.tobytes(), fmt
        assert np.array_equal(bits(cost), bits(wcost)), fmt


@pytest.mark.parametrize("pin", [False, True])
def test_mine_host_record_buffer_too_small(pin):
    """A record buffer smaller than the result fails with BM_ELIMIT (no overrun)."""
    from paper_1509_08639_b200 import hostapi, synth

    sc = synth.make_corpus(*synth.c2_shape(400), seed=13)
    model = bm.load_model(golden("model5k_fwd.json"))
    pb = hostapi.PinnedBatch(sc.packed, sc.world.packed_lexicon(), pin=pin, wire=True)
    _, k, _ = hostapi.mine_pinned(pb, model, 0.5, 0.2)
    assert k > 10
    pb.rec_cap = k - 1
    guard = pb.rec[k - 1:].copy()
    with pytest.raises(bm.ResourceLimitError):
        hostapi.mine_pinned(pb, model, 0.5, 0.2)
    assert pb.rec[k - 1:].tobytes() == guard.tobytes()


# ---------------------------------------------------------------- tuning
@pytest.mark.parametrize("docs,tfile,k,grid", [
    ("docs40.jsonl", "tune10.json", 10, None),
    ("docs10_noisy.jsonl", "tune_noisy.json", 10, None),
    ("docs10_noisy.jsonl", "tune_noisy_small.json", 3, ([0.3, 0.6], [0.1, 0.4])),
])
def test_tune_matches_reference(world500, docs, tfile, k, grid):
    lex, fwd, _ = world500
    raw = load_docs(docs)[:k]
    dev = bm.GoldSet(docs=pairs_of(raw), gold=[{(i, j) for i, j in d["gold"]} for d in raw])
    kw = {} if grid is None else {"thresholds": grid[0], "penalties": grid[1]}
    got = bm.tune(fwd, lex, dev, **kw)
    assert bm.tune_result_to_json(got) == open(golden(tfile)).read()


@pytest.mark.parametrize("docs,tfile,k,grid", [
    ("docs40.jsonl", "tune10.json", 10, None),
    ("docs10_noisy.jsonl", "tune_noisy.json", 10, None),
    ("docs10_noisy.jsonl", "tune_noisy_small.json", 3, ([0.3, 0.6], [0.1, 0.4])),
])
def test_tune_file_native_gold_path(world500, tmp_path, docs, tfile, k, grid):
    """tune_file == tune(load_gold_set(path)) with the gold set read and its keys
    packed natively: the reference's trace bytes."""
    from paper_1509_08639_b200.ingest import NativeCorpus

    lex, fwd, _ = world500
    path = str(tmp_path / "gold.jsonl")
    with open(path, "w") as fh:
        for d in load_docs(docs)[:k]:
            fh.write(json.dumps(d) + "\n")
    assert NativeCorpus.load(path, gold=True) is not None
    kw = {} if grid is None else {"thresholds": grid[0], "penalties": grid[1]}
    got = bm.tune_file(path, fwd, lex, **kw)
    assert bm.tune_result_to_json(got) == open(golden(tfile)).read()


def test_tune_file_errors_match_load_gold_set(world500, tmp_path):
    """Files the reference rejects take the Python path and raise its errors."""
    lex, fwd, _ = world500
    good = load_docs("docs10_noisy.jsonl")[:3]
    cases = {
        "bounds": [dict(good[0], gold=[[0, 0], [999, 1]])],
        "missing": [{k: v for k, v in good[0].items() if k != "gold"}],
        "entries": [dict(good[0], gold=[[0, 1.5]])],
        "empty": [dict(good[0], tgt=[])],
    }
    for name, docs in cases.items():
        path = str(tmp_path / f"{name}.jsonl")
        with open(path, "w") as fh:
            for d in docs:
                fh.write(json.dumps(d) + "\n")
        with pytest.raises(bm.DataError) as a:
            bm.load_gold_set(path)
        with pytest.raises(bm.DataError) as b:
            bm.tune_file(path, fwd, lex)
        assert str(a.value) == str(b.value)


def test_tune_synthetic_vs_oracle(oracle_mod):
    from paper_1509_08639_b200 import engine, synth

    sc = synth.make_corpus(*synth.c2_shape(48), seed=12)
    model = bm.load_model(golden("model5k_fwd.json"))
    plex = sc.world.packed_lexicon()
    pens = [0.05, 0.1, 0.2, 0.3, 0.4, 0.6, 0.8, 1.6]
    thrs = [0.2, 0.3, 0.4, 0.5, 0.6, 0.7, 0.8, 0.9]
    keys = [np.asarray(g[:, 0] * int(sc.packed.m[d]) + g[:, 1], np.int64) for d, g in enumerate(sc.gold)]
    p, h = engine.tune_counts(engine.DeviceCorpus.upload(sc.packed), engine.DeviceLexicon.upload(plex),
                              engine.DocView.of(sc.packed), model, pens, thrs, keys)
    wp, wh = oracle_mod.tune(oracle_mod.HostBatch(sc.packed, plex), model, pens, thrs, keys, threads=8)
    assert np.array_equal(p, wp) and np.array_equal(h, wh)


@pytest.mark.parametrize("n_pen", [1, 2, 3, 4, 7, 9])
def test_tune_multi_penalty_passes_vs_oracle(oracle_mod, n_pen):
    """Penalties run in passes of 4 / 2 / 1 through nw_band_kernel<D, NP>;
    mixed sizes (multi-band docs hand boundary rows per penalty), ties from a
    repeated penalty, and 0.0 (every diagonal wins) == oracle counts."""
    from paper_1509_08639_b200 import engine

    sc = _synth_mixed(9)
    model = bm.load_model(golden("model5k_fwd.json"))
    plex = sc.world.packed_lexicon()
    pens = [0.2, 0.0, 0.6, 0.2, 1.6, 0.05, 0.35, 0.9, 0.1][:n_pen]
    thrs = [0.3, 0.5, 0.8]
    keys = [np.asarray(g[:, 0] * int(sc.packed.m[d]) + g[:, 1], np.int64) for d, g in enumerate(sc.gold)]
    p, h = engine.tune_counts(engine.DeviceCorpus.upload(sc.packed), engine.DeviceLexicon.upload(plex),
                              engine.DocView.of(sc.packed), model, pens, thrs, keys)
    wp, wh = oracle_mod.tune(oracle_mod.HostBatch(sc.packed, plex), model, pens, thrs, keys, threads=8)
    assert np.array_equal(p, wp) and np.array_equal(h, wh)


@pytest.mark.parametrize("run", ["2", "7", "32"])
def test_tune_runs_of_single_band_documents_vs_oracle(oracle_mod, monkeypatch, run):
    """nw_seq_kernel: runs of single-band documents laid end to end (forced run
    lengths; n from 1 to 128, m from 1 to 300 incl. m < 4 and m % 4 != 0, with
    multi-band documents between runs), 8 penalties incl. 0 and inf in passes of
    4, 8 thresholds: pred / hit counts == oracle."""
    from paper_1509_08639_b200 import engine, synth

    monkeypatch.setenv("BM_NW_SEQ_RUN", run)
    r = np.random.default_rng(77)
    D = 160
    n = r.integers(1, 129, D)
    m = r.integers(1, 301, D)
    n[:8] = [1, 128, 127, 4, 3, 100, 300, 129]
    m[:8] = [1, 1, 3, 300, 5, 100, 200, 64]
    n[40::37] = r.integers(129, 400, len(n[40::37]))  # multi-band documents between runs
    g = np.minimum(n, m) // 2
    sc = synth.make_corpus(g, n - g, m - g, vocab=2000, seed=31)
    model = bm.load_model(golden("model5k_fwd.json"))
    plex = sc.world.packed_lexicon()
    pens = [0.05, 0.0, 0.2, float("inf"), 0.4, 0.6, 0.8, 1.6]
    thrs = [0.2, 0.3, 0.4, 0.5, 0.6, 0.7, 0.8, 0.9]
    keys = [np.asarray(gd[:, 0] * int(sc.packed.m[d]) + gd[:, 1], np.int64) for d, gd in enumerate(sc.gold)]
    p, h = engine.tune_counts(engine.DeviceCorpus.upload(sc.packed), engine.DeviceLexicon.upload(plex),
                              engine.DocView.of(sc.packed), model, pens, thrs, keys)
    wp, wh = oracle_mod.tune(oracle_mod.HostBatch(sc.packed, plex), model, pens, thrs, keys, threads=8)
    assert np.array_equal(p, wp) and np.array_equal(h, wh)


def test_sharded_mining_equals_single(oracle_mod):
    """Two LPT shards mined separately (as two ranks would) == one batch."""
    from paper_1509_08639_b200 import engine, shard, synth

    sc = _synth_mixed(7)
    model = bm.load_model(golden("model5k_fwd.json"))
    plex = sc.world.packed_lexicon()
    parts = [shard.mine_shard(sc.packed, plex, model, 0.5, 0.2, r, 2)[0] for r in range(2)]
    got = shard.restore_order(parts)
    want, _ = oracle_mod.mine(oracle_mod.HostBatch(sc.packed, plex), model, 0.5, 0.2, threads=8)
    assert got.tobytes() == want.tobytes()


def test_device_bidirectional_merge_edge_cases():
    """bm_merge_bidir against bidirectional_merge (miner.py:131-155) on random
    paths over documents with repeated sentences (equal normalized keys),
    confidence ties between and within directions, and swapped passes."""
    from paper_1509_08639_b200 import engine, miner
    from paper_1509_08639_b200.pack import Packer

    rng = np.random.default_rng(77)
    words = ["alpha", "beta", "Gamma", "gamma", "delta"]
    pairs, fw, bw, sf, sb = [], [], [], [], []
    for d in range(60):
        n, m = int(rng.integers(1, 12)), int(rng.integers(1, 12))
        src = [" ".join(rng.choice(words, 2)) + "." for _ in range(n)]
        tgt = [" ".join(rng.choice(words, 2)) + "." for _ in range(m)]
        pairs.append(bm.parse_document_pair({"id": f"d{d}", "src_lang": "xx", "tgt_lang": "yy",
                                             "src": src, "tgt": tgt}, "mem", d + 1))
        for out, swap in ((fw, sf), (bw, sb)):
            s = bool(rng.integers(0, 2))
            swap.append(s)
            a, b = (m, n) if s else (n, m)  # the pass's own orientation
            i = j = 0
            recs = []
            while i < a and j < b:  # a random monotone path's diagonal cells
                if rng.random() < 0.6:
                    c = float(rng.choice([0.5, 0.75, 0.9, rng.random()]))
                    recs.append((d, i, j, c))
                i += int(rng.integers(1, 3))
                j += int(rng.integers(1, 3))
            out.extend(recs)

    def to_arr(rs):
        a = np.zeros(len(rs), dtype=np.dtype(engine.N.RECORD_DTYPE))
        for q, (d, i, j, c) in enumerate(rs):
            a[q] = (d, i, j, 0, c)
        return a

    F, B = to_arr(fw), to_arr(bw)
    pk = Packer()
    for p in pairs:
        pk.add_pair(p)
    corpus = pk.finish()
    dev = engine.device()
    import torch

    fd = torch.from_numpy(F.view(np.uint8).copy()).to(dev)
    bd = torch.from_numpy(B.view(np.uint8).copy()).to(dev)
    got = engine.merge_bidir(fd, len(F), bd, len(B), corpus.src0, corpus.tgt0,
                             engine.to_dev(corpus.norm_key, dev), sf, sb)
    by_doc = miner._split_by_doc(got, len(pairs))
    for d, p in enumerate(pairs):
        want = miner.bidirectional_merge(
            miner._records_to_pairs(p, F[F["doc"] == d], sf[d]),
            miner._records_to_pairs(p, B[B["doc"] == d], sb[d]))
        have = miner._merged_to_pairs(p, by_doc[d])
        assert [(r.src_index, r.tgt_index, r.confidence, r.direction) for r in have] == \
            [(r.src_index, r.tgt_index, r.confidence, r.direction) for r in want]


@pytest.mark.parametrize("chunk", [4096, 65536])
def test_mine_corpus_file_streams_in_chunks(world500, tmp_path, monkeypatch, chunk):
    """Chunked mine_corpus_file (ingest, mine, merge, emit per chunk; the next
    chunk read meanwhile): the reference's 1,000-document TSV bytes and report
    for any chunk size."""
    import gzip

    from paper_1509_08639_b200 import ingest

    lex, fwd, bwd = world500
    p = str(tmp_path / "docs1000.jsonl")
    with gzip.open(golden("docs1000_s77.jsonl.gz"), "rb") as fi, open(p, "wb") as fo:
        fo.write(fi.read())
    monkeypatch.setenv("BM_STREAM_CHUNK_BYTES", str(chunk))
    sink = io.StringIO()
    rep = bm.mine_corpus_file(p, fwd, bwd, lex, bm.MinerConfig(bm.MiningParams(0.5, 0.2)), sink)
    want = json.load(open(golden("mine1000_bi.json")))
    text = sink.getvalue()
    assert ingest.LAST_TIMINGS["chunks"] > 3
    assert text.count("\n") == want["lines"]
    assert hashlib.sha256(text.encode()).hexdigest() == want["sha256"]
    ref = io.StringIO()
    rrep = bm.mine_corpus(bm.load_document_pairs(p), fwd, bwd, lex,
                          bm.MinerConfig(bm.MiningParams(0.5, 0.2)), ref)
    rep.wall_clock_seconds = rrep.wall_clock_seconds = 0.0
    assert bm.report_to_json(rep) == bm.report_to_json(rrep)


def test_mine_corpus_file_hands_the_rest_to_python_mid_file(world500, tmp_path, monkeypatch):
    """A document the native path cannot take (a direction the models do not
    know, then invalid UTF-8) in a later chunk: earlier chunks are mined
    natively, the rest by the Python reader -- the same bytes and error as
    mine_corpus(load_document_pairs(path))."""
    lex, fwd, bwd = world500
    docs = load_docs("docs40.jsonl")
    bad = dict(docs[30], src_lang="zz")
    lines = [json.dumps(d) + "\n" for d in docs[:30]] + [json.dumps(bad) + "\n"] + \
            [json.dumps(d) + "\n" for d in docs[31:]]
    monkeypatch.setenv("BM_STREAM_CHUNK_BYTES", "2048")
    for tail in (b"", b"\xff\xfe not utf-8\n"):
        p = str(tmp_path / f"mixed{len(tail)}.jsonl")
        with open(p, "wb") as fh:
            fh.write("".join(lines).encode())
            fh.write(tail)
        cfg = bm.MinerConfig(bm.MiningParams(0.5, 0.2))
        outs, errs = [], []
        for fn in (lambda o: bm.mine_corpus_file(p, fwd, bwd, lex, cfg, o),
                   lambda o: bm.mine_corpus(bm.load_document_pairs(p), fwd, bwd, lex, cfg, o)):
            o = io.StringIO()
            try:
                fn(o)
                errs.append(None)
            except Exception as exc:  # noqa: BLE001 -- compared below
                errs.append((type(exc), str(exc)))
            outs.append(o.getvalue())
        assert outs[0] == outs[1] and outs[0].count("\n") > 100
        assert errs[0] == errs[1] and errs[0] is not None


def test_trim_releases_scratch_and_mining_continues(oracle_mod):
    """bm_trim drops the per-stream workspaces; the next calls regrow them and
    give the same records."""
    from paper_1509_08639_b200 import _native, engine, synth

    g, a, b = synth.c3_shape(300, seed=12)
    sc = synth.make_corpus_native(g, a, b, seed=12)
    model = bm.load_model(golden("model5k_fwd.json"))
    dc = engine.DeviceCorpus.upload(sc.packed)
    dl = engine.DeviceLexicon.upload(sc.world.packed_lexicon())
    view = engine.DocView.of(sc.packed)
    first, _ = engine.mine(dc, dl, view, model, 0.5, 0.2)
    assert _native.lib().bm_trim() == 0
    again, _ = engine.mine(dc, dl, view, model, 0.5, 0.2)
    assert first.tobytes() == again.tobytes()


def test_tune_pinned_chunks_equal_device_sweep():
    """hostapi.tune_pinned (chunked H2D overlapping per-chunk bm_tune, counts
    added across chunks) gives the device-resident sweep's counts exactly, for
    several chunk counts, including chunks of one document."""
    from paper_1509_08639_b200 import engine, hostapi, synth

    sc = synth.make_corpus(*synth.c3_shape(300, seed=77), seed=77)
    c = sc.packed
    model = bm.load_model(golden("model5k_fwd.json"))
    plex = sc.world.packed_lexicon()
    dl = engine.DeviceLexicon.upload(plex)
    keys = [np.asarray(gd[:, 0] * int(c.m[d]) + gd[:, 1], np.int64) for d, gd in enumerate(sc.gold)]
    pens, thrs = [0.05, 0.2, 0.4, 1.6, 0.1], [0.3, 0.5, 0.7]
    want_p, want_h = engine.tune_counts(engine.DeviceCorpus.upload(c), dl, engine.DocView.of(c),
                                        model, pens, thrs, keys)
    gk, goff = engine.pack_gold(keys)
    tp = hostapi.TunePinned(c, gk, goff)
    for k in (1, 3, 7, 300):
        p, h = hostapi.tune_pinned(tp, dl, model, pens, thrs, n_chunks=k)
        assert np.array_equal(p, want_p) and np.array_equal(h, want_h), k
