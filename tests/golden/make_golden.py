"""Generate the golden fixtures from the REFERENCE implementation.

Run in the build container only (needs /root/reference, read-only):

    python tests/golden/make_golden.py

Everything written here is produced by /root/reference/pkg/src/bimine (and its
test generator tests/synthgen.py) on seeded inputs; the test-suite compares the
CPU oracle and the GPU kernels against these files. The GPU box never reads
/root/reference.
"""

from __future__ import annotations

import gzip
import hashlib
import io
import itertools
import json
import math
import os
import random
import struct
import sys

import numpy as np

REF = "/root/reference/pkg"
sys.path[:0] = [os.path.join(REF, "src"), os.path.join(REF, "tests")]

import synthgen  # noqa: E402  (reference test generator)
from bimine.aligner import (  # noqa: E402
    SimilarityMatrix,
    build_similarity_matrix,
    nw_align,
)
from bimine.classifier import SCHEMA_ID, ClassifierModel, model_to_json, train  # noqa: E402
from bimine.corpus import (  # noqa: E402
    SeedCorpus,
    Sentence,
    load_seed_corpus,
    normalize,
    parse_document_pair,
    segment_sentences,
    tokenize,
)
from bimine.lexicon import Lexicon, load_lexicon  # noqa: E402
from bimine.miner import MinerConfig, MiningParams, mine_corpus, report_to_json  # noqa: E402
from bimine.tuner import GoldSet, tune, tune_result_to_json  # noqa: E402

OUT = os.path.dirname(os.path.abspath(__file__))
TMP = "/tmp/bimine_golden"
os.makedirs(TMP, exist_ok=True)


def w(name: str) -> str:
    return os.path.join(OUT, name)


def bits(x: float) -> int:
    return struct.unpack("<Q", struct.pack("<d", x))[0]


def ops_of(path) -> np.ndarray:
    return np.array([{"D": 0, "GS": 1, "GT": 2}[mv.op] for mv in path.moves], dtype=np.int8)


def save_dp(name: str, mats_paths_costs) -> None:
    ops = [ops_of(p) for _, p in mats_paths_costs]
    off = np.zeros(len(ops) + 1, dtype=np.int64)
    off[1:] = np.cumsum([len(o) for o in ops])
    np.savez_compressed(
        w(name),
        ops=np.concatenate(ops) if ops else np.zeros(0, np.int8),
        off=off,
        cost=np.array([p.total_cost for _, p in mats_paths_costs], dtype=np.float64),
        shape=np.array([m.shape for m, _ in mats_paths_costs], dtype=np.int64).reshape(-1, 2),
    )


def world(vocab_size: int, tag: str):
    vocab = synthgen.make_vocab(vocab_size)
    lex_path = w(f"lex{tag}.tsv")
    synthgen.write_lexicon_tsv(lex_path, vocab)
    lex = load_lexicon(lex_path, synthgen.SRC_LANG, synthgen.TGT_LANG)
    pairs = synthgen.make_seed_corpus(2000, vocab, seed=11, noise=0.1)
    src, tgt = os.path.join(TMP, f"seed{tag}.src"), os.path.join(TMP, f"seed{tag}.tgt")
    synthgen.write_seed_files(pairs, src, tgt)
    seed = load_seed_corpus(src, tgt)
    fwd = train(seed, lex, seed=42)
    swapped = SeedCorpus(pairs=[(t, s) for s, t in seed.pairs], dropped=seed.dropped)
    bwd = train(swapped, lex.reversed(), seed=43)
    for name, model in (("fwd", fwd), ("bwd", bwd)):
        with open(w(f"model{tag}_{name}.json"), "w") as fh:
            fh.write(model_to_json(model))
    return vocab, lex, fwd, bwd


def write_docs(name: str, docs: list[dict], gz: bool = False) -> None:
    buf = io.StringIO()
    for d in docs:
        buf.write(json.dumps(d, sort_keys=True) + "\n")
    data = buf.getvalue().encode("utf-8")
    if gz:
        with gzip.GzipFile(w(name), "wb", mtime=0) as fh:
            fh.write(data)
    else:
        with open(w(name), "wb") as fh:
            fh.write(data)


def mine_text(pairs, fwd, bwd, lex, t=0.5, p=0.2):
    sink = io.StringIO()
    rep = mine_corpus(iter(pairs), fwd, bwd, lex, MinerConfig(params=MiningParams(t, p)), sink)
    rep.wall_clock_seconds = 0.0
    return sink.getvalue(), report_to_json(rep)


def stack_matrices(name: str, mats: list[np.ndarray]) -> None:
    np.savez_compressed(
        w(name),
        flat=np.concatenate([m.ravel() for m in mats]),
        shape=np.array([m.shape for m in mats], dtype=np.int64),
    )


def main() -> None:
    # 1. exp: the glibc exp CPython calls (classifier.py:100-104)
    rng = np.random.default_rng(5)
    zs = np.concatenate([
        rng.uniform(-40, 40, 12000), rng.uniform(-745, 0, 3000), rng.uniform(-1e-10, 1e-10, 500),
        -np.abs(rng.standard_normal(3000)) * 3, np.array([0.0, -0.0, -1e-300, -708.4, -745.2,
                                                          -1000.0, -512.0, -511.9, 1e-17]),
    ])
    ex = np.array([bits(math.exp(float(z))) for z in zs], dtype=np.uint64)
    np.savez_compressed(w("exp_golden.npz"), z=zs, exp_bits=ex)

    # 2. corpus semantics (tokenize / normalize / segmentation)
    samples = [
        "Hello, world! 3.14 apples", "Dr. Smith went to Washington. He said no.",
        "It's a_b test -- done?! Yes. 2024 was fine.", "Ünïcödé Straße ﬁne ÅNGSTRÖM 　tab\there",
        "école  CAFÉ ²³ ١٢٣ ⅨⅩ", "etc. is not an end. Mr. X. Next one", "   ", "",
        "one.Two three. four", "Wait... What? 5 o'clock!",
    ]
    corpus_gold = {
        "tokens": {s: tokenize(s) for s in samples},
        "normalized": {s: normalize(s) for s in samples},
        "segments": {s: [x.raw for x in segment_sentences(s)] for s in samples},
    }
    with open(w("corpus_golden.json"), "w", encoding="utf-8") as fh:
        json.dump(corpus_gold, fh, ensure_ascii=False, indent=1, sort_keys=True)

    # 3. the reference test world (conftest.py: 500 words, seeds 11/42/43/21)
    vocab, lex, fwd, bwd = world(500, "500")
    docs40 = synthgen.make_comparable_corpus(40, vocab, seed=21, noise=0.1)
    write_docs("docs40.jsonl", docs40)
    pairs40 = [parse_document_pair(d, "mem", i) for i, d in enumerate(docs40, 1)]
    stack_matrices("S40.npz", [build_similarity_matrix(p, fwd, lex).cells for p in pairs40])
    txt, rep = mine_text(pairs40, fwd, None, lex)
    open(w("mine40_fwd.tsv"), "w").write(txt)
    open(w("mine40_fwd.report.json"), "w").write(rep)
    txt, rep = mine_text(pairs40, fwd, bwd, lex)
    open(w("mine40_bi.tsv"), "w").write(txt)
    open(w("mine40_bi.report.json"), "w").write(rep)
    txt, _ = mine_text(pairs40, fwd, bwd, lex, t=0.3, p=0.05)
    open(w("mine40_bi_t03_p005.tsv"), "w").write(txt)
    dev = GoldSet(docs=pairs40[:10], gold=[{(i, j) for i, j in d["gold"]} for d in docs40[:10]])
    open(w("tune10.json"), "w").write(tune_result_to_json(tune(fwd, lex, dev)))

    # acceptance #4 shape: 1000 docs, seed 77, bidirectional, 0.5 / 0.2
    docs1k = synthgen.make_comparable_corpus(1000, vocab, seed=77, noise=0.1)
    write_docs("docs1000_s77.jsonl.gz", docs1k, gz=True)
    pairs1k = [parse_document_pair(d, "mem", i) for i, d in enumerate(docs1k, 1)]
    txt, rep = mine_text(pairs1k, fwd, bwd, lex)
    json.dump({"sha256": hashlib.sha256(txt.encode()).hexdigest(), "lines": txt.count("\n"),
               "report": json.loads(rep)}, open(w("mine1000_bi.json"), "w"), indent=1)

    # acceptance #6 shape: noisy dev set, default grid
    noisy = synthgen.make_comparable_corpus(10, vocab, seed=33, noise=0.4)
    write_docs("docs10_noisy.jsonl", noisy)
    devn = GoldSet(docs=[parse_document_pair(d, "mem", i) for i, d in enumerate(noisy, 1)],
                   gold=[{(i, j) for i, j in d["gold"]} for d in noisy])
    open(w("tune_noisy.json"), "w").write(tune_result_to_json(tune(fwd, lex, devn)))
    small = GoldSet(docs=devn.docs[:3], gold=devn.gold[:3])
    open(w("tune_noisy_small.json"), "w").write(
        tune_result_to_json(tune(fwd, lex, small, thresholds=[0.3, 0.6], penalties=[0.1, 0.4])))

    # 4. the 5k-word world of the benchmark configs (C1: 200 x 200)
    vocab5k, lex5k, fwd5k, bwd5k = world(5000, "5k")
    rng_py = random.Random(2026)
    c1 = synthgen.make_comparable_doc("c1", vocab5k, rng_py, n_gold=120, n_src_distract=80,
                                      n_tgt_distract=80, noise=0.1)
    write_docs("doc200.jsonl", [c1])
    p200 = parse_document_pair(c1, "mem", 1)
    S200 = build_similarity_matrix(p200, fwd5k, lex5k).cells
    np.savez_compressed(w("S200.npz"), S=S200)
    txt, rep = mine_text([p200], fwd5k, None, lex5k)
    open(w("mine200_fwd.tsv"), "w").write(txt)
    txt, rep = mine_text([p200], fwd5k, bwd5k, lex5k)
    open(w("mine200_bi.tsv"), "w").write(txt)
    docs100 = synthgen.make_comparable_corpus(6, vocab5k, seed=4, noise=0.1, n_gold=60,
                                              n_src_distract=40, n_tgt_distract=40)
    write_docs("docs100x6.jsonl", docs100)
    pairs100 = [parse_document_pair(d, "mem", i) for i, d in enumerate(docs100, 1)]
    txt, _ = mine_text(pairs100, fwd5k, bwd5k, lex5k)
    open(w("mine100x6_bi.tsv"), "w").write(txt)

    # 5. stress scoring: unicode, digits, punctuation, case, multi-candidate
    #    lexicon with duplicates / absent candidates / non-positive probabilities
    rs = random.Random(99)
    words_s = ["hund", "Katze", "maus", "Über", "straße", "ÉCOLE", "x", "ab", "Ab", "ﬁne"]
    words_t = ["dog", "cat", "mouse", "over", "street", "school", "y", "ba", "BA", "fine", "pup"]
    extras = [".", ",", "!", "?", "--", "_", "'", "2020", "1999", "42", "²", "٣", "3.5"]

    def sent(words):
        k = rs.randint(0, 9)
        toks = [rs.choice(words + extras) for _ in range(k)]
        return " ".join(toks) if rs.random() < 0.9 else "".join(toks)

    stress_docs = []
    for k in range(12):
        n, m = rs.randint(1, 9), rs.randint(1, 9)
        stress_docs.append({"id": f"s{k}", "src_lang": "aa", "tgt_lang": "bb",
                            "src": [sent(words_s) for _ in range(n)] or ["x"],
                            "tgt": [sent(words_t) for _ in range(m)] or ["y"]})
    entries = {
        "hund": [("dog", 0.9), ("pup", 0.5), ("hound", 0.4)],
        "katze": [("cat", 0.8), ("cat", 0.3)],
        "maus": [("mouse", 0.0), ("mice", 0.7)],
        "über": [("over", 1.0), ("above", 0.2)],
        "straße": [("street", 0.6), ("road", 0.6)],
        "école": [("school", 0.9), ("ba", 0.1)],
        "ab": [("ba", 0.5), ("y", 0.5)],
        "x": [("y", -0.5), ("ba", 0.3)],
        "ﬁne": [("fine", 0.9)],
        "2020": [("2020", 0.9)],
        "notinanydoc": [("dog", 0.9)],
    }
    slex = Lexicon(direction=("aa", "bb"), entries=entries)
    smodel = ClassifierModel(SCHEMA_ID, [0.7, 2.5, -1.25, 0.5, -0.75, 1.5, 0.125], -0.3,
                             ("aa", "bb"), 0.5, 0.2)
    spairs = [parse_document_pair(d, "mem", i) for i, d in enumerate(stress_docs, 1)]
    stack_matrices("S_stress.npz", [build_similarity_matrix(p, smodel, slex).cells for p in spairs])
    write_docs("docs_stress.jsonl", stress_docs)
    json.dump({"direction": list(slex.direction), "entries": {k: [list(c) for c in v]
               for k, v in entries.items()}}, open(w("lex_stress.json"), "w"), indent=1)
    open(w("model_stress.json"), "w").write(model_to_json(smodel))

    # 6. DP golden vectors (matrices regenerated from the same numpy seeds)
    dp = []
    grid = [0.0, 0.25, 0.5, 0.75, 1.0]
    for vals in itertools.product(grid, repeat=4):
        S = np.array(vals).reshape(2, 2)
        for p in (0.05, 0.25, 0.5, 1.0):
            dp.append((S, nw_align(SimilarityMatrix(S), p)))
    save_dp("dp_grid2x2.npz", dp)
    r = np.random.default_rng(202)
    dp = []
    for _ in range(200):
        n, m = r.integers(1, 51, size=2)
        S = r.random((n, m))
        p = float(r.uniform(0.05, 1.0))
        dp.append((S, nw_align(SimilarityMatrix(S), p)))
    save_dp("dp_s202.npz", dp)
    r = np.random.default_rng(12)
    dp = [(S, nw_align(SimilarityMatrix(S), 0.3)) for S in
          (r.random((127, 129)), r.random((128, 128)), r.random((130, 257)))]
    save_dp("dp_s12_tiles.npz", dp)
    r = np.random.default_rng(7)
    dp = []
    for _ in range(60):  # quantized values: many exact ties (tie order D > GS > GT)
        n, m = r.integers(1, 40, size=2)
        S = r.integers(0, 5, size=(n, m)) / 4.0
        p = float(r.choice([0.0, 0.125, 0.25, 0.5, 1.0]))
        dp.append((S, nw_align(SimilarityMatrix(S), p)))
    save_dp("dp_quantized.npz", dp)
    r = np.random.default_rng(303)
    S = r.random((2000, 2000))
    save_dp("dp_s303_2000.npz", [(S, nw_align(SimilarityMatrix(S), 0.3))])
    r = np.random.default_rng(31)
    dp = []
    for n, m in [(300, 40), (40, 300), (129, 1), (1, 129), (256, 257), (513, 200), (700, 700)]:
        S = r.random((n, m))
        dp.append((S, nw_align(SimilarityMatrix(S), 0.2)))
    save_dp("dp_s31_shapes.npz", dp)
    print("golden fixtures written to", OUT)


if __name__ == "__main__":
    main()
