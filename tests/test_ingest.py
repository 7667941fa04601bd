"""Native corpus path (csrc/bm_ingest.cpp, ingest.py) vs the Python reader.

Host-only: ingestion, lexicon lowering and TSV emission run without a GPU, so
these parity checks are CPU tests. The GPU round trip (mine_corpus_file ==
mine_corpus(load_document_pairs(...))) is in test_gpu_parity.py.
"""

import gzip
import json
import os
import unicodedata

import numpy as np
import pytest

import paper_1509_08639_b200 as bm
from paper_1509_08639_b200 import _native as N
from paper_1509_08639_b200.aligner import MinedPair
from paper_1509_08639_b200.corpus import load_document_pairs, tokenize
from paper_1509_08639_b200.ingest import NativeCorpus
from paper_1509_08639_b200.miner import bidirectional_merge, format_pair_line
from paper_1509_08639_b200.pack import pack_lexicon, pack_pairs

from conftest import golden

FIELDS = ("n_tok", "n_punct", "n_alpha", "tok_off", "tok_id", "tok_alpha", "dig_off", "dig_id",
          "src0", "n", "tgt0", "m")

EDGE_LINES = [
    # segmentation: abbreviations, digits after a period, ! and ?, trailing spaces
    {"id": "e1", "src_lang": "xx", "tgt_lang": "yy",
     "src": "Dr. Smith met Mr. Jones at 5 p.m. today! Was it 2019? 42 is the answer.  ",
     "tgt": ["a b", "   ", "C-d e_f g__h", "x\tyz"]},
    # escapes, punctuation-only tokens, mixed case, digit tokens, underscores
    {"id": 7, "src_lang": "yy", "tgt_lang": "xx", "src": ["HELLO, World!!", "abc123 4567 _x_"],
     "tgt": "Line one.\nLine Two.\tEnd.\r\nno. 5 etc. Vs. X", "extra": {"a": [1, 2.5e3, None, True]}},
    # empty side: dropped at load (reported), nothing interned
    {"id": "empty", "src_lang": "xx", "tgt_lang": "yy", "src": "   ", "tgt": ["kept"]},
    {"id": "empty2", "src_lang": "xx", "tgt_lang": "yy", "src": ["a"], "tgt": []},
    # duplicate keys: the last one wins
    {"id": "dup", "src_lang": "xx", "tgt_lang": "yy", "src": "first", "tgt": "T"},
]


def write_jsonl(path, lines, raw_extra=(), newline="\n"):
    with open(path, "w", newline="") as fh:
        for obj in lines:
            fh.write(json.dumps(obj) + newline)
        for raw in raw_extra:
            fh.write(raw + newline)


def python_side(path):
    skipped = []
    pairs = list(load_document_pairs(path, on_skip=lambda pid, why: skipped.append((pid, why))))
    return pairs, pack_pairs(pairs), skipped


def assert_same_pack(nc, pc):
    for f in FIELDS:
        a, b = getattr(nc.packed, f), getattr(pc, f)
        assert a.shape == b.shape and np.array_equal(a, b), f
    assert nc.n_ids == len(pc.strings)


@pytest.fixture(scope="module")
def lex():
    return bm.load_lexicon(golden("lex5k.tsv"), "xx", "yy")


@pytest.mark.parametrize("name", ["docs40.jsonl", "doc200.jsonl", "docs10_noisy.jsonl",
                                  "docs100x6.jsonl", "docs_stress.jsonl"])
def test_ingest_matches_python_packer(name, lex):
    path = golden(name)
    nc = NativeCorpus.load(path)
    assert nc is not None
    pairs, pc, skipped = python_side(path)
    assert_same_pack(nc, pc)
    assert nc.doc_ids == [p.id for p in pairs]
    assert nc.langs == [(p.source.lang, p.target.lang) for p in pairs]
    assert [(pid, f"empty {side} document") for _l, pid, side in nc.skipped] == skipped
    pl, nl = pack_lexicon(lex, pc), nc.lexicon(lex)
    for f in ("fwd_off", "fwd_cand", "rev_off", "rev_cand"):
        assert np.array_equal(getattr(pl, f), getattr(nl, f)), f


def test_ingest_edge_cases(tmp_path, lex):
    p = str(tmp_path / "edge.jsonl")
    raw = ['{"id": "dup", "src_lang": "xx", "tgt_lang": "yy", "src": "first", "src": ["second one", "x"], "tgt": "t", "tgt": "U V."}',
           "   \t",
           '{"id": 12, "src_lang": "xx", "tgt_lang": "yy", "src": ["\\u0041b\\/c"], "tgt": ["q\\\\r"]}']
    write_jsonl(p, EDGE_LINES, raw, newline="\r\n")
    nc = NativeCorpus.load(p)
    assert nc is not None
    pairs, pc, skipped = python_side(p)
    assert_same_pack(nc, pc)
    assert nc.doc_ids == [x.id for x in pairs]
    assert [(pid, f"empty {side} document") for _l, pid, side in nc.skipped] == skipped
    assert len(skipped) == 2


def test_ingest_bare_cr_lines(tmp_path):
    p = str(tmp_path / "cr.jsonl")
    write_jsonl(p, EDGE_LINES[:2], newline="\r")
    nc = NativeCorpus.load(p)
    pairs, pc, _ = python_side(p)
    assert_same_pack(nc, pc)


@pytest.mark.parametrize("line", [
    # text NFC would change or that lowercases outside the per-character map
    '{"id": "u", "src_lang": "xx", "tgt_lang": "yy", "src": "cafe\\u0301", "tgt": "x"}',  # e + acute
    '{"id": "u", "src_lang": "xx", "tgt_lang": "yy", "src": "cafe\u0301", "tgt": "x"}',
    '{"id": "u", "src_lang": "xx", "tgt_lang": "yy", "src": "a\u0316\u0317", "tgt": "x"}',  # 2 marks
    '{"id": "u", "src_lang": "xx", "tgt_lang": "yy", "src": "\u212a", "tgt": "x"}',  # Kelvin sign
    '{"id": "u", "src_lang": "xx", "tgt_lang": "yy", "src": "ΟΔΟΣ", "tgt": "x"}',  # final sigma
    '{"id": "u", "src_lang": "xx", "tgt_lang": "yy", "src": ["x"], "tgt": ["İstanbul"]}',  # 2-cp lower
    '{"id": "u", "src_lang": "xx", "tgt_lang": "yy", "src": "\\ud800", "tgt": "x"}',  # lone surrogate
    '{"id": "u", "src_lang": "xx", "tgt_lang": "yy", "src": "\\udc00\\ud800", "tgt": "x"}',
    '{"id": "a\\u0000b", "src_lang": "xx", "tgt_lang": "yy", "src": "a", "tgt": "b"}',  # NUL id
    '{"id": 1.5, "src_lang": "xx", "tgt_lang": "yy", "src": "a", "tgt": "b"}',          # float id
    '{"id": "a", "src_lang": "xx", "tgt_lang": "xx", "src": "a", "tgt": "b"}',          # same langs
    '{"id": "a", "src_lang": "xx", "src": "a", "tgt": "b"}',                           # missing
    '{"id": "a", "src_lang": "xx", "tgt_lang": "yy", "src": [1], "tgt": "b"}',          # bad item
    '{"id": "a", "src_lang": "xx", "tgt_lang": "yy", "src": "a", "tgt": "b"',           # truncated
    '{"id": "a", "src_lang": "xx", "tgt_lang": "yy", "src": "a", "tgt": "b", "x": NaN}',
    '["not", "an", "object"]',
])
def test_ingest_declines_outside_the_subset(tmp_path, line):
    p = str(tmp_path / "bad.jsonl")
    with open(p, "w", encoding="utf-8") as fh:
        fh.write(line + "\n")
    assert NativeCorpus.load(p) is None


@pytest.mark.parametrize("raw", [b"\xff", b"\xc0\x80", b"\xed\xa0\x80", b"\xf4\x90\x80\x80",
                                 b"\xe2\x82"])
def test_ingest_declines_invalid_utf8(tmp_path, raw):
    p = tmp_path / "bad.jsonl"
    p.write_bytes(b'{"id": "u", "src_lang": "xx", "tgt_lang": "yy", "src": "a' + raw +
                  b'", "tgt": "x"}\n')
    assert NativeCorpus.load(str(p)) is None


UNICODE_LINES = [
    {"id": "pl-1", "src_lang": "xx", "tgt_lang": "yy",
     "src": "Zażółć gęślą jaźń. Źdźbło trawy! Ósmy dzień? 3 koty. ŁÓDŹ i GDAŃSK. dr. Żak, prof. Łuk.",
     "tgt": ["Grüße aus Köln.", "ÉCOLE élève. Ça va!", "Straße ẞ MASSE"]},
    {"id": "ελ", "src_lang": "yy", "tgt_lang": "xx",
     "src": "Καλημέρα κόσμε. Η ΑΘΗΝΑ είναι 3η! Ρωσικά: Привет, МИР. Ёлка.",
     "tgt": "漢字かな交じり文。カタカナ．ＡＢＣ１２３ and ٣٤٥ and ²³ ½ Ⅻ ǅungla ǈ."},
    {"id": 42, "src_lang": "xx", "tgt_lang": "yy",
     "src": "nbsp\u00a0here.\u2003Em space\u3000ideographic\u2028line\u0085nel x\u200bzw.",
     "tgt": ["emoji 😀🎉 ok", "😀 escaped pair", "\u00a0\u2003", "tab\there"]},
    {"id": "m", "src_lang": "xx", "tgt_lang": "yy",
     "src": "a\u0316b mark alone \u0316 x. Ünï. Mr. Ø. DR. X. Vs. Y. \u0130 no",
     "tgt": "ǅ titlecase. ǈ. Ⅻ roman. ℌ script. 𝐀 bold. ᾈ greek"},
]


def test_ingest_unicode_matches_python_packer(tmp_path, lex):
    """Non-ASCII text the native path accepts reproduces Python's tokenizer,
    NFC/lower/split normalizer and segmentation exactly (Polish, German,
    Greek, Cyrillic, CJK, Unicode spaces and digits, astral characters)."""
    p = str(tmp_path / "uni.jsonl")
    lines = [dict(x) for x in UNICODE_LINES]

    def write():  # odd lines as \\u escapes (surrogate pairs for astral chars)
        with open(p, "w", encoding="utf-8") as fh:
            for q, obj in enumerate(lines):
                fh.write(json.dumps(obj, ensure_ascii=bool(q % 2)) + "\n")

    write()
    # İ (U+0130) lowercases to two code points: that file is Python's
    assert NativeCorpus.load(p) is None
    lines[3]["src"] = lines[3]["src"].replace("\u0130", "I")
    write()
    nc = NativeCorpus.load(p)
    assert nc is not None
    pairs, pc, skipped = python_side(p)
    assert any(ord(ch) > 0xFFFF for pr in pairs for s in pr.target.sentences for ch in s.raw)
    assert_same_pack(nc, pc)
    assert nc.doc_ids == [x.id for x in pairs]
    assert nc.langs == [(x.source.lang, x.target.lang) for x in pairs]
    pl, nl = pack_lexicon(lex, pc), nc.lexicon(lex)
    for f in ("fwd_off", "fwd_cand", "rev_off", "rev_cand"):
        assert np.array_equal(getattr(pl, f), getattr(nl, f)), f
    # emission: raw sentences and ids go out as UTF-8, unique tokens counted
    nd = pc.n_docs
    z = np.zeros(nd, dtype=np.uint8)
    recs = np.array([(d, i, j, 0, 0.75) for d in range(nd) for i in range(int(pc.n[d]))
                     for j in range(int(pc.m[d])) if (i + j) % 2 == 0],
                    dtype=np.dtype(N.RECORD_DTYPE))
    data, rep = nc.emit(recs, None, z, z, z)
    want = []
    for k in range(nd):
        pr = pairs[k]
        src, tgt = pr.source.sentences, pr.target.sentences
        want += [MinedPair(src[int(r["i"])], tgt[int(r["j"])], 0.75, pr.id, "forward", int(r["i"]),
                           int(r["j"])) for r in recs[recs["doc"] == k]]
    assert data.decode("utf-8") == "".join(format_pair_line(r) for r in want)
    st, tt = set(), set()
    for r in want:
        st.update(tokenize(r.src.normalized))
        tt.update(tokenize(r.tgt.normalized))
    assert rep[:5] == [len(want), len(want), 0, len(st), len(tt)]


def _random_text(rng, pool, n):
    return "".join(pool[int(x)] for x in rng.integers(0, len(pool), n))


def test_ingest_unicode_fuzz_accept_implies_identical(tmp_path):
    """Random text over a wide code-point pool (letters, marks, spaces, digits,
    punctuation, astral, case-special characters): whenever the native reader
    accepts a file, its packing equals Python's; it accepts most of the
    NFC-stable, simply-lowercased pool."""
    rng = np.random.default_rng(11)
    wide = [chr(c) for c in list(range(0x20, 0x7f)) + list(range(0xa0, 0x250)) +
            list(range(0x300, 0x370)) + list(range(0x370, 0x530)) + list(range(0x1e00, 0x1f00)) +
            list(range(0x2000, 0x2070)) + list(range(0x2150, 0x2190)) + list(range(0x3000, 0x3040)) +
            list(range(0xac00, 0xac40)) + list(range(0x1100, 0x1180)) + list(range(0xff00, 0xff60)) +
            [0x1d400, 0x1f600, 0x10400, 0x10428, 0x130, 0x3a3, 0x212a, 0x2126, 0x85, 0x1c, 0x1f]
            if not 0xd800 <= c <= 0xdfff and c not in (0x22, 0x5c)]
    def simple(ch):  # NFC-stable starter, one-code-point lower of the same classes
        lo = ch.lower()
        return (unicodedata.normalize("NFC", ch) == ch and unicodedata.combining(ch) == 0
                and not 0x1161 <= ord(ch) <= 0x11c2 and ch != "\u03a3" and len(lo) == 1
                and (lo.isalnum(), lo.isspace()) == (ch.isalnum(), ch.isspace()))

    safe = [ch for ch in wide if (ch.isalnum() or ch.isspace() or ch in ".!?,;:-") and simple(ch)]
    accepted = 0
    for trial in range(60):
        pool = wide if trial % 2 else safe
        lines = []
        for d in range(4):
            src = ". ".join(_random_text(rng, pool, 12) for _ in range(3))
            lines.append({"id": f"f{trial}-{d}", "src_lang": "xx", "tgt_lang": "yy", "src": src,
                          "tgt": [_random_text(rng, pool, 10), _random_text(rng, pool, 6) + "."]})
        p = str(tmp_path / f"fz{trial}.jsonl")
        with open(p, "w", encoding="utf-8") as fh:
            for obj in lines:
                fh.write(json.dumps(obj, ensure_ascii=bool(trial % 3 == 0)) + "\n")
        nc = NativeCorpus.load(p)
        if nc is None:
            continue
        accepted += 1
        pairs, pc, skipped = python_side(p)
        assert_same_pack(nc, pc)
        assert nc.doc_ids == [x.id for x in pairs]
        assert [(pid, f"empty {side} document") for _l, pid, side in nc.skipped] == skipped
    assert accepted >= 20


def _fake_records(pc, seed, dirn):
    """Plausible mined records: per doc some diagonal cells with quantized
    confidences (ties exercise the merge rules)."""
    rng = np.random.default_rng(seed)
    rows = []
    for d in range(pc.n_docs):
        n, m = int(pc.n[d]), int(pc.m[d])
        k = min(n, m)
        for i in range(k):
            if rng.random() < 0.6:
                rows.append((d, i, min(m - 1, i + (dirn and rng.random() < 0.2)), 0,
                             round(rng.random() * 4) / 4 * 0.5 + 0.5))
    return np.array(rows, dtype=np.dtype(N.RECORD_DTYPE))


def test_emit_matches_python_merge_and_format(tmp_path):
    path = golden("docs40.jsonl")
    nc = NativeCorpus.load(path)
    pairs, pc, _ = python_side(path)
    nd = pc.n_docs
    rng = np.random.default_rng(3)
    sw_f = (rng.random(nd) < 0.3).astype(np.uint8)
    sw_b = 1 - sw_f
    skip = (rng.random(nd) < 0.1).astype(np.uint8)
    fwd = _fake_records(pc, 1, 0)
    bwd = _fake_records(pc, 2, 1)

    def to_pairs(k, recs, swapped):
        pair = pairs[k]
        src, tgt = pair.source.sentences, pair.target.sentences
        out = []
        for r in recs[recs["doc"] == k]:
            i, j, c = int(r["i"]), int(r["j"]), float(r["conf"])
            if swapped:  # records index the oriented pair (source = pair.target)
                i, j = j, i
            if i >= len(src) or j >= len(tgt):
                continue
            out.append(MinedPair(src[i], tgt[j], c, pair.id, "backward" if swapped else "forward",
                                 i, j))
        return out

    # records must index the oriented pair: drop the ones a swap makes invalid
    def valid(recs, sw):
        keep = []
        for r in recs:
            d, i, j = int(r["doc"]), int(r["i"]), int(r["j"])
            n, m = int(pc.n[d]), int(pc.m[d])
            if sw[d]:
                n, m = m, n
            keep.append(i < n and j < m)
        return recs[np.array(keep, dtype=bool)]

    fwd, bwd = valid(fwd, sw_f), valid(bwd, sw_b)
    for has_bwd in (False, True):
        data, rep = nc.emit(fwd, bwd if has_bwd else None, sw_f, sw_b, skip)
        want = []
        for k in range(nd):
            if skip[k]:
                continue
            mined = to_pairs(k, fwd, sw_f[k])
            if has_bwd:
                mined = bidirectional_merge(mined, to_pairs(k, bwd, sw_b[k]))
            want.extend(mined)
        text = "".join(format_pair_line(r) for r in want)
        assert data.decode("ascii") == text
        src_tok, tgt_tok = set(), set()
        for r in want:
            src_tok.update(tokenize(r.src.normalized))
            tgt_tok.update(tokenize(r.tgt.normalized))
        assert rep == [len(want), sum(r.direction == "forward" for r in want),
                       sum(r.direction == "backward" for r in want), len(src_tok), len(tgt_tok),
                       int((skip == 0).sum())]


@pytest.fixture(scope="module")
def docs1000(tmp_path_factory):
    p = str(tmp_path_factory.mktemp("c") / "docs1000.jsonl")
    with gzip.open(golden("docs1000_s77.jsonl.gz"), "rb") as fi, open(p, "wb") as fo:
        fo.write(fi.read())
    return p, python_side(p)


@pytest.mark.parametrize("threads", ["1", "3", "7", "16"])
def test_ingest_1000_doc_corpus_any_thread_count(docs1000, threads, monkeypatch):
    """Chunks parsed in parallel re-intern into the sequential id order."""
    monkeypatch.setenv("BM_INGEST_THREADS", threads)
    p, (_, pc, _) = docs1000
    nc = NativeCorpus.load(p)
    assert nc is not None
    assert_same_pack(nc, pc)


def test_emit_on_a_multi_chunk_ingest(docs1000, monkeypatch):
    """Merge keys are chunk-local: the merge must still match Python's."""
    monkeypatch.setenv("BM_INGEST_THREADS", "5")
    p, (pairs, pc, _) = docs1000
    nc = NativeCorpus.load(p)
    nd = pc.n_docs
    fwd = _fake_records(pc, 4, 0)
    bwd = _fake_records(pc, 5, 1)
    z = np.zeros(nd, dtype=np.uint8)
    data, rep = nc.emit(fwd, bwd, z, z, z)
    want = []
    for k in range(nd):
        pair = pairs[k]
        src, tgt = pair.source.sentences, pair.target.sentences
        f = [MinedPair(src[int(r["i"])], tgt[int(r["j"])], float(r["conf"]), pair.id, "forward",
                       int(r["i"]), int(r["j"])) for r in fwd[fwd["doc"] == k]]
        b = [MinedPair(src[int(r["i"])], tgt[int(r["j"])], float(r["conf"]), pair.id, "forward",
                       int(r["i"]), int(r["j"])) for r in bwd[bwd["doc"] == k]]
        want.extend(bidirectional_merge(f, b))
    assert data.decode("ascii") == "".join(format_pair_line(r) for r in want)
    assert rep[0] == len(want)


def test_emit_thread_count_invariance(docs1000, monkeypatch):
    """Document ranges formatted on separate threads concatenate to the same
    bytes and the same unique-token counts as one thread."""
    p, (pairs, pc, _) = docs1000
    fwd = _fake_records(pc, 6, 0)
    bwd = _fake_records(pc, 7, 1)
    z = np.zeros(pc.n_docs, dtype=np.uint8)
    skip = (np.random.default_rng(8).random(pc.n_docs) < 0.05).astype(np.uint8)
    got = []
    for threads in ("1", "3", "8", "32"):
        monkeypatch.setenv("BM_INGEST_THREADS", threads)
        nc = NativeCorpus.load(p)
        got.append(nc.emit(fwd, bwd, z, z, skip))
        got.append(nc.emit(fwd, None, z, z, skip))
    assert all(g == got[0] for g in got[0::2]) and all(g == got[1] for g in got[1::2])
    assert got[0][1][0] > 1000


def test_ingest_empty_and_missing_files(tmp_path):
    p = tmp_path / "empty.jsonl"
    p.write_bytes(b"")
    nc = NativeCorpus.load(str(p))
    assert nc is not None and nc.packed.n_docs == 0 and nc.n_ids == 0
    p.write_bytes(b"\n  \n\t\n")
    nc = NativeCorpus.load(str(p))
    assert nc is not None and nc.packed.n_docs == 0
    # the Python reader raises the reference's error for a missing file
    assert NativeCorpus.load(str(tmp_path / "missing.jsonl")) is None


def test_native_gold_set_keys(tmp_path):
    """bm_ingest_gold_jsonl: per-document ascending unique keys i * m + j equal
    to load_gold_set's cells; files load_gold_set rejects are declined."""
    import json

    from conftest import golden, load_docs
    from paper_1509_08639_b200.ingest import NativeCorpus

    docs = load_docs("docs10_noisy.jsonl")
    docs[1]["gold"] = docs[1]["gold"] + docs[1]["gold"][:2]  # duplicates: a set
    path = str(tmp_path / "gold.jsonl")
    with open(path, "w") as fh:
        for d in docs:
            fh.write(json.dumps(d) + "\n")
    nc = NativeCorpus.load(path, gold=True)
    assert nc is not None
    dev = bm.load_gold_set(path)
    for d, cells in enumerate(dev.gold):
        m = len(dev.docs[d].target.sentences)
        want = sorted(i * m + j for i, j in cells)
        got = nc.gold_keys[nc.gold_off[d] : nc.gold_off[d + 1]].tolist()
        assert got == want
    for bad in ([dict(docs[0], gold=[[0, True]])], [dict(docs[0], gold=[[-1, 0]])],
                [{k: v for k, v in docs[0].items() if k != "gold"}], []):
        p = str(tmp_path / "bad.jsonl")
        with open(p, "w") as fh:
            for d in bad:
                fh.write(json.dumps(d) + "\n")
        assert NativeCorpus.load(p, gold=True) is None
