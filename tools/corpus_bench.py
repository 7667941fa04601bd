"""End-to-end corpus mining from a JSONL file.

Writes a C2-shaped corpus (N docs of 100x100 synthetic sentences, the synth
world's 5k-word dictionary) as JSONL, then times
  python: mine_corpus(load_document_pairs(path), ...)   (Python reader/packer)
  native: mine_corpus_file(path, ...)                  (C++ reader, GPU, C++ TSV)
with the forward and backward models, and checks the TSV outputs are equal.
Usage: python tools/corpus_bench.py [N_DOCS] [--no-python]
"""
import io
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import paper_1509_08639_b200 as bm  # noqa: E402
from paper_1509_08639_b200 import synth  # noqa: E402


def main():
    n_docs = int(sys.argv[1]) if len(sys.argv) > 1 and sys.argv[1].isdigit() else 10000
    path = f"/tmp/c2_{n_docs}.jsonl"
    sc = synth.make_corpus(*synth.c2_shape(n_docs), seed=21)
    lex = sc.world.lexicon()
    if not os.path.exists(path):
        t0 = time.perf_counter()
        with open(path, "w") as fh:
            for a in range(0, n_docs, 1000):
                for p in sc.doc_pairs(range(a, min(n_docs, a + 1000))):
                    fh.write(json.dumps({"id": p.id, "src_lang": p.source.lang,
                                         "tgt_lang": p.target.lang,
                                         "src": [s.raw for s in p.source.sentences],
                                         "tgt": [s.raw for s in p.target.sentences]}) + "\n")
        print(json.dumps({"wrote": path, "s": time.perf_counter() - t0}), flush=True)
    fwd = bm.load_model(os.path.join(ROOT, "tests", "golden", "model5k_fwd.json"))
    bwd = bm.load_model(os.path.join(ROOT, "tests", "golden", "model5k_bwd.json"))
    cfg = bm.MinerConfig(bm.MiningParams(0.5, 0.2))
    res = {"docs": n_docs, "bytes": os.path.getsize(path)}
    # warm up the device path once
    bm.mine_corpus_file(path, fwd, bwd, lex, cfg, io.StringIO())
    t0 = time.perf_counter()
    out_n = io.StringIO()
    rep = bm.mine_corpus_file(path, fwd, bwd, lex, cfg, out_n)
    res["native_s"] = time.perf_counter() - t0
    res["native_docs_per_s"] = n_docs / res["native_s"]
    res["pairs"] = rep.pairs_emitted
    from paper_1509_08639_b200.ingest import LAST_TIMINGS
    res["native_phases_s"] = {k: round(v, 4) for k, v in LAST_TIMINGS.items()}
    if "--no-python" not in sys.argv:
        t0 = time.perf_counter()
        out_p = io.StringIO()
        bm.mine_corpus(bm.load_document_pairs(path), fwd, bwd, lex, cfg, out_p)
        res["python_s"] = time.perf_counter() - t0
        res["python_docs_per_s"] = n_docs / res["python_s"]
        res["identical"] = out_p.getvalue() == out_n.getvalue()
    print(json.dumps(res), flush=True)


if __name__ == "__main__":
    main()
