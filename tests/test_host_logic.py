"""Host-side logic of the drop-in (no GPU): input contract, validation and
error behaviour, merge rules, formatting and loaders. Cases follow the
reference's unit tests (pkg/tests/test_*.py) so behaviour matches call for call."""

import json
import math

import numpy as np
import pytest

import paper_1509_08639_b200 as bm
from conftest import golden, load_docs, pairs_of
from paper_1509_08639_b200.pack import Packer, pack_lexicon, pack_pairs


# ----------------------------------------------------------------- corpus
def test_tokenize_normalize_segment_match_reference():
    gold = json.load(open(golden("corpus_golden.json"), encoding="utf-8"))
    for s, toks in gold["tokens"].items():
        assert bm.tokenize(s) == toks
    for s, norm in gold["normalized"].items():
        assert bm.normalize(s) == norm
    for s, segs in gold["segments"].items():
        assert [x.raw for x in bm.segment_sentences(s)] == segs


def test_parse_document_pair_errors():
    with pytest.raises(bm.DataError, match="missing field 'tgt'"):
        bm.parse_document_pair({"id": 1, "src_lang": "a", "tgt_lang": "b", "src": []}, "p", 3)
    with pytest.raises(bm.DataError, match="must differ"):
        bm.parse_document_pair({"id": 1, "src_lang": "a", "tgt_lang": "a", "src": [], "tgt": []}, "p", 1)
    with pytest.raises(bm.DataError, match="string or a list"):
        bm.parse_document_pair({"id": 1, "src_lang": "a", "tgt_lang": "b", "src": 3, "tgt": []}, "p", 1)


def test_load_document_pairs_skips_empty_sides(tmp_path):
    p = tmp_path / "d.jsonl"
    p.write_text(json.dumps({"id": "a", "src_lang": "x", "tgt_lang": "y", "src": [], "tgt": ["B."]}) + "\n"
                 + json.dumps({"id": "b", "src_lang": "x", "tgt_lang": "y", "src": ["A."], "tgt": ["B."]}) + "\n")
    skipped = []
    got = list(bm.load_document_pairs(str(p), on_skip=lambda i, r: skipped.append((i, r))))
    assert [d.id for d in got] == ["b"] and skipped == [("a", "empty src document")]


# ----------------------------------------------------------------- lexicon
def test_lexicon_reverse_cache_and_max_prob(tmp_path):
    p = tmp_path / "l.tsv"
    p.write_text("# c\nHund\tdog\t0.5\nhund\tDOG\t0.9\nwolf\tdog\t0.3\n")
    lex = bm.load_lexicon(str(p), "de", "en")
    assert lex.entries == {"hund": [("dog", 0.9)], "wolf": [("dog", 0.3)]}
    rev = lex.reversed()
    assert rev.entries == {"dog": [("hund", 0.9), ("wolf", 0.3)]}
    assert lex.reversed() is rev and rev.reversed() is lex
    assert rev.direction == ("en", "de")


@pytest.mark.parametrize("line,msg", [("a\tb\n", "3 tab"), ("a\tb\tx\n", "bad probability"),
                                       ("a\tb\t1.5\n", "outside"), ("a\tb\tnan\n", "outside"),
                                       (" \tb\t0.5\n", "empty word")])
def test_load_lexicon_errors(tmp_path, line, msg):
    p = tmp_path / "l.tsv"
    p.write_text(line)
    with pytest.raises(bm.DataError, match=msg):
        bm.load_lexicon(str(p))


# ----------------------------------------------------------------- classifier
def test_load_model_validation(tmp_path):
    good = json.load(open(golden("model500_fwd.json")))
    m = bm.load_model(golden("model500_fwd.json"))
    assert m.weights == good["weights"] and m.direction == ("xx", "yy")
    for patch, msg in (({"version": 2}, "unsupported"), ({"weights": [1.0]}, "requires 7"),
                       ({"default_threshold": 2.0}, "out of range")):
        p = tmp_path / "m.json"
        p.write_text(json.dumps({**good, **patch}))
        with pytest.raises(bm.DataError, match=msg):
            bm.load_model(str(p))
    p = tmp_path / "bad.json"
    p.write_text("{")
    with pytest.raises(bm.DataError, match="not a valid model"):
        bm.load_model(str(p))


def test_model_json_round_trip(tmp_path):
    m = bm.load_model(golden("model5k_fwd.json"))
    p = tmp_path / "m.json"
    bm.save_model(m, str(p))
    assert open(p).read() == open(golden("model5k_fwd.json")).read()


def test_confidence_schema_mismatch_names_both():
    model = bm.ClassifierModel("pairwise-v1", [0.0] * 7, 0.0, ("a", "b"), 0.5, 0.2)
    with pytest.raises(bm.DataError, match="other-v9.*pairwise-v1"):
        bm.confidence(model, bm.FeatureVector(values=[0.0] * 7, schema_id="other-v9"))


def test_train_is_out_of_scope():
    with pytest.raises(NotImplementedError, match="reference"):
        bm.train(None, None)


# ----------------------------------------------------------------- aligner types
def test_similarity_matrix_validation(monkeypatch):
    with pytest.raises(ValueError, match="2-D"):
        bm.SimilarityMatrix(np.array([0.5, 0.5]))
    with pytest.raises(ValueError, match=r"\[0, 1\]"):
        bm.SimilarityMatrix(np.array([[1.2]]))
    with pytest.raises(ValueError):
        bm.SimilarityMatrix(np.array([[float("nan")]]))
    monkeypatch.setattr("paper_1509_08639_b200.aligner.MAX_CELLS", 16)
    with pytest.raises(bm.ResourceLimitError, match="cell limit"):
        bm.SimilarityMatrix(np.zeros((5, 5)) + 0.5)
    bm.SimilarityMatrix(np.zeros((4, 4)) + 0.5)


def test_mining_params_and_penalty_validation():
    with pytest.raises(ValueError, match="threshold"):
        bm.MiningParams(1.0001, 0.2)
    with pytest.raises(ValueError, match="penalty"):
        bm.MiningParams(0.5, -0.2)
    with pytest.raises(ValueError, match="penalty"):
        bm.nw_align(bm.SimilarityMatrix(np.eye(2)), -0.5)
    with pytest.raises(ValueError, match="workers"):
        bm.nw_align_wavefront(bm.SimilarityMatrix(np.eye(2)), 0.2, workers=0)
    with pytest.raises(ValueError, match="unknown engine"):
        bm.run_engine("quantum", bm.SimilarityMatrix(np.eye(2)), 0.2)


def test_build_similarity_matrix_checks_before_gpu(world500, monkeypatch):
    lex, fwd, _ = world500
    pair = pairs_of(load_docs("docs40.jsonl"))[0]
    other = bm.ClassifierModel("pairwise-v1", [0.0] * 7, 0.0, ("aa", "bb"), 0.5, 0.2)
    with pytest.raises(bm.DataError, match="does not match document"):
        bm.build_similarity_matrix(pair, other, lex)
    monkeypatch.setattr("paper_1509_08639_b200.aligner.MAX_CELLS", 4)
    with pytest.raises(bm.ResourceLimitError, match="cell limit"):
        bm.build_similarity_matrix(pair, fwd, lex)


# ----------------------------------------------------------------- miner host logic
def test_miner_config_validation():
    p = bm.MiningParams(0.5, 0.2)
    with pytest.raises(ValueError, match="workers"):
        bm.MinerConfig(p, workers=0)
    with pytest.raises(ValueError, match="wavefront_workers"):
        bm.MinerConfig(p, wavefront_workers=0)
    with pytest.raises(ValueError, match="unknown engine"):
        bm.MinerConfig(p, engine="x")


def _mp(src, tgt, conf, doc="d", direction="forward", si=0, tj=0):
    return bm.MinedPair(bm.Sentence.from_text(src), bm.Sentence.from_text(tgt), conf, doc,
                        direction, si, tj)


def test_bidirectional_merge_rules():
    # test_miner.py:127-183
    fwd = [_mp("a", "x", 0.9), _mp("b", "y", 0.8, si=1)]
    bwd = [_mp("a", "x", 0.95, direction="backward"), _mp("b", "y", 0.8, direction="backward", si=1),
           _mp("c", "z", 0.7, direction="backward", si=2)]
    out = bm.bidirectional_merge(fwd, bwd)
    assert [(r.src.raw, r.direction, r.confidence) for r in out] == [
        ("a", "backward", 0.95), ("b", "forward", 0.8), ("c", "backward", 0.7)]
    # exact tie between two backward records: first seen stays
    t = bm.bidirectional_merge([], [_mp("A", "x", 0.5, direction="backward", si=1),
                                    _mp("a", "X", 0.5, direction="backward", si=0)])
    assert len(t) == 1 and t[0].src.raw == "A"


def test_format_pair_line_sanitizes():
    rec = _mp("a\tb", "c\nd", 0.1234567, doc="id\r1", direction="backward")
    assert bm.format_pair_line(rec) == "a b\tc d\t0.123457\tid 1\tbackward\n"


def test_mine_document_direction_errors_raise_before_gpu(world500):
    lex, fwd, _ = world500
    pair = pairs_of(load_docs("docs40.jsonl"))[0]
    cfg = bm.MinerConfig(bm.MiningParams(0.5, 0.2))
    other = bm.ClassifierModel("pairwise-v1", [0.0] * 7, 0.0, ("aa", "bb"), 0.5, 0.2)
    with pytest.raises(bm.DataError, match="matches neither"):
        bm.mine_document(pair, other, lex, cfg)
    with pytest.raises(bm.DataError, match="lexicon direction"):
        bm.mine_document(pair, fwd, lex.reversed(), cfg)


def test_mine_documents_stops_at_first_error(world500):
    lex, fwd, _ = world500
    pairs = pairs_of(load_docs("docs40.jsonl"))[:3]
    bad = bm.DocumentPair("bad", bm.Document("bad", "qq", pairs[0].source.sentences),
                          bm.Document("bad", "rr", pairs[0].target.sentences))
    empty = bm.DocumentPair("e", bm.Document("e", "xx", []), pairs[0].target)
    # empty side -> skip reason; direction mismatch -> error after the docs before it
    res, err = bm.miner.mine_documents([empty, bad] + pairs, fwd, None, lex,
                                       bm.MinerConfig(bm.MiningParams(0.5, 0.2)))
    assert isinstance(err, bm.DataError) and "matches neither" in str(err)
    assert res == [([], "document pair 'e': empty src side")]


def test_report_json_shape():
    r = bm.MiningReport(pairs_emitted=3, docs_processed=2)
    d = json.loads(bm.report_to_json(r))
    assert d["per_direction"] == {"forward": 0, "backward": 0} and d["pairs_emitted"] == 3


# ----------------------------------------------------------------- tuner host logic
def test_f_measure_cases():
    assert bm.f_measure(set(), set()) == (1.0, 1.0, 1.0)
    assert bm.f_measure({(1,)}, {(2,)}) == (0.0, 0.0, 0.0)
    p, r, f = bm.f_measure({("a",), ("b",)}, {("a",), ("b",), ("c",), ("d",)})
    assert (p, r) == (1.0, 0.5) and f == pytest.approx(2 / 3)
    assert bm.f_measure(set(), {(1,)}) == (0.0, 0.0, 0.0)


def test_tune_validation_before_gpu(world500):
    lex, fwd, _ = world500
    raw = load_docs("docs40.jsonl")[:2]
    dev = bm.GoldSet(docs=pairs_of(raw), gold=[{(i, j) for i, j in d["gold"]} for d in raw])
    with pytest.raises(bm.DataError, match="empty"):
        bm.tune(fwd, lex, bm.GoldSet(docs=[], gold=[]))
    with pytest.raises(ValueError, match="grid"):
        bm.tune(fwd, lex, dev, thresholds=[])
    with pytest.raises(ValueError, match="threshold"):
        bm.tune(fwd, lex, dev, thresholds=[1.5])
    with pytest.raises(ValueError, match="penalty"):
        bm.tune(fwd, lex, dev, penalties=[-0.2])
    with pytest.raises(ValueError, match="out of bounds"):
        bm.GoldSet(docs=dev.docs[:1], gold=[{(99, 0)}])


def test_load_gold_set(tmp_path):
    p = tmp_path / "g.jsonl"
    p.write_text(json.dumps({"id": "a", "src_lang": "x", "tgt_lang": "y", "src": ["A."], "tgt": ["B."],
                             "gold": [[0, 0]]}) + "\n")
    gs = bm.load_gold_set(str(p))
    assert gs.gold == [{(0, 0)}]
    p.write_text(json.dumps({"id": "a", "src_lang": "x", "tgt_lang": "y", "src": ["A."], "tgt": ["B."],
                             "gold": [[0, 5]]}) + "\n")
    with pytest.raises(bm.DataError, match="out of"):
        bm.load_gold_set(str(p))


# ----------------------------------------------------------------- packing
def test_packer_sets_and_multiplicities():
    pk = Packer()
    s = bm.Sentence.from_text("Hund hund HUND 2020, 7 x_y.")
    pk.add_sentence(s)
    c = pk.finish()
    toks = dict(zip((c.strings[i] for i in c.tok_id), c.tok_alpha.tolist()))
    assert toks["hund"] == 3 and toks["2020"] == 0 and toks[","] == 0 and toks["x"] == 1
    assert int(c.n_tok[0]) == len(s.tokens) and int(c.n_alpha[0]) == 5  # hund x3, x, y
    assert int(c.n_punct[0]) == 3  # "," "_" "."
    assert sorted(c.strings[i] for i in c.dig_id) == ["2020", "7"]


def test_pack_lexicon_keeps_only_present_candidates(world500):
    lex, _, _ = world500
    corpus = pack_pairs(pairs_of(load_docs("docs40.jsonl"))[:2])
    pl = pack_lexicon(lex, corpus)
    assert pl.fwd_off.shape[0] == len(corpus.strings) + 1
    for k, s in enumerate(corpus.strings):
        cands = {corpus.strings[c] for c in pl.fwd_cand[pl.fwd_off[k]:pl.fwd_off[k + 1]]}
        want = {c for c, _ in lex.entries.get(s, []) if c in corpus.ids}
        assert cands == want


def test_doc_token_max_matches_loop():
    corpus = pack_pairs(pairs_of(load_docs("docs_stress.jsonl")))
    am = corpus.doc_token_max()
    for d in range(corpus.n_docs):
        s = corpus.n_tok[corpus.src0[d]:corpus.src0[d] + corpus.n[d]].tolist()
        t = corpus.n_tok[corpus.tgt0[d]:corpus.tgt0[d] + corpus.m[d]].tolist()
        assert am[d] == max(s + t + [0])
