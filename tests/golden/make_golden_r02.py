"""Round-2 golden fixtures, produced by the REFERENCE implementation.

Run in the build container only (needs /root/reference, read-only):

    python tests/golden/make_golden_r02.py

mine40_badline.{tsv,json}: docs40.jsonl with a malformed line after its first
5 documents, mined by the reference's mine_corpus(load_document_pairs(path))
with workers=1 (lazy map: the 5 documents are written, then the loader's
DataError propagates, miner.py:236-237) and workers=3 (pool.map submits every
document first, so nothing is written, miner.py:238-245).
"""

from __future__ import annotations

import io
import json
import os
import sys

REF = "/root/reference/pkg"
sys.path[:0] = [os.path.join(REF, "src"), os.path.join(REF, "tests")]

from bimine.classifier import load_model  # noqa: E402
from bimine.corpus import load_document_pairs  # noqa: E402
from bimine.errors import DataError  # noqa: E402
from bimine.lexicon import load_lexicon  # noqa: E402
from bimine.miner import MinerConfig, MiningParams, mine_corpus  # noqa: E402

OUT = os.path.dirname(os.path.abspath(__file__))
TMP = "/tmp/bimine_golden_r02"
os.makedirs(TMP, exist_ok=True)


def badline_corpus(path: str) -> None:
    lines = open(os.path.join(OUT, "docs40.jsonl"), encoding="utf-8").read().splitlines(True)
    with open(path, "w", encoding="utf-8") as fh:
        fh.writelines(lines[:5])
        fh.write("{not json\n")
        fh.writelines(lines[5:])


def big_token_docs() -> list[dict]:
    """docs40[0], a doc whose first sentences hold 70,003 / 66,002 tokens (one
    alphabetic token repeated 70,000 / 66,000 times, so both the multiplicity
    and the hit counts exceed 16 bits), and docs40[2]."""
    docs = [json.loads(x) for x in open(os.path.join(OUT, "docs40.jsonl"), encoding="utf-8")][:3]
    big = dict(docs[1], id="big")
    big["src"] = ["waaa " * 70000 + "wadf walb."] + docs[1]["src"][1:]
    big["tgt"] = ["vaaa " * 66000 + "vadf vafr."] + docs[1]["tgt"][1:]
    return [docs[0], big, docs[2]]


def main() -> None:
    lex = load_lexicon(os.path.join(OUT, "lex500.tsv"), "xx", "yy")
    fwd = load_model(os.path.join(OUT, "model500_fwd.json"))
    bwd = load_model(os.path.join(OUT, "model500_bwd.json"))
    path = os.path.join(TMP, "bad.jsonl")
    badline_corpus(path)
    result = {}
    for workers in (1, 3):
        sink = io.StringIO()
        try:
            mine_corpus(load_document_pairs(path), fwd, bwd, lex,
                        MinerConfig(MiningParams(0.5, 0.2), workers=workers), sink)
            err = None
        except DataError as exc:
            err = str(exc).replace(path, "<path>")
        result[f"workers{workers}"] = {"error": err, "tsv": sink.getvalue()}
    with open(os.path.join(OUT, "mine40_badline.json"), "w") as fh:
        json.dump(result, fh, indent=1)
    print({k: (v["error"], len(v["tsv"])) for k, v in result.items()})

    # sentences longer than 65,535 tokens, mined by the reference
    from bimine.corpus import parse_document_pair
    from bimine.miner import report_to_json

    pairs = [parse_document_pair(d, "mem", i) for i, d in enumerate(big_token_docs(), 1)]
    sink = io.StringIO()
    rep = mine_corpus(iter(pairs), fwd, bwd, lex, MinerConfig(MiningParams(0.5, 0.2)), sink)
    rep.wall_clock_seconds = 0.0
    text = sink.getvalue()
    import hashlib

    out = {"lines": text.count("\n"), "sha256": hashlib.sha256(text.encode()).hexdigest(),
           "report": report_to_json(rep),
           "short_lines": [ln for ln in text.splitlines(True) if len(ln) < 400]}
    with open(os.path.join(OUT, "mine_big_tokens.json"), "w") as fh:
        json.dump(out, fh, indent=1)
    print("big tokens:", out["lines"], "lines", len(out["short_lines"]), "short")


if __name__ == "__main__":
    main()
