"""The reference's acceptance criteria for the hot path, run through this
package on the GPU (bimine tests/test_acceptance.py #1 and #5).

#1: the DP's optimal cost equals an exhaustive enumeration of every alignment
path (all 2x2 matrices over the grid {0, .25, .5, .75, 1} x 4 penalties, and
1,000 random 4x4 grid matrices, seed 404), to 1e-9 like the reference.
#5: mining with both models yields at least the forward-only pairs on the
40-document fixture, and strictly more on a constructed document that only
the backward model accepts.
"""

import io
import itertools
from functools import lru_cache

import numpy as np
import pytest

import paper_1509_08639_b200 as bm
from paper_1509_08639_b200.classifier import SCHEMA_ID, ClassifierModel
from paper_1509_08639_b200.corpus import parse_document_pair

from conftest import golden

pytestmark = pytest.mark.gpu

GRID = (0.0, 0.25, 0.5, 0.75, 1.0)


@lru_cache(maxsize=None)
def all_paths(n: int, m: int) -> tuple:
    """Every monotone alignment path from (0, 0) to (n, m) as a tuple of moves
    ("D", i, j) / ("GS", i) / ("GT", j)."""
    if n == 0 and m == 0:
        return ((),)
    out = []
    if n > 0 and m > 0:
        out += [p + (("D", n - 1, m - 1),) for p in all_paths(n - 1, m - 1)]
    if n > 0:
        out += [p + (("GS", n - 1),) for p in all_paths(n - 1, m)]
    if m > 0:
        out += [p + (("GT", m - 1),) for p in all_paths(n, m - 1)]
    return tuple(out)


def brute_min_cost(S: np.ndarray, p: float) -> float:
    best = float("inf")
    for path in all_paths(*S.shape):
        c = 0.0
        for mv in path:
            c += (1.0 - S[mv[1], mv[2]]) if mv[0] == "D" else p
        best = min(best, c)
    return best


def test_01_alignment_cost_matches_brute_force():
    assert len(all_paths(4, 4)) == 321  # Delannoy number D(4, 4)
    cases = []
    for vals in itertools.product(GRID, repeat=4):
        for p in (0.05, 0.25, 0.5, 1.0):
            cases.append((np.array(vals).reshape(2, 2), p))
    rng = np.random.default_rng(404)
    for _ in range(1000):
        S = rng.choice(GRID, size=(4, 4))
        cases.append((S, float(rng.choice([0.05, 0.1, 0.3, 0.7, 1.2]))))
    by_p: dict[float, list[int]] = {}
    for k, (_, p) in enumerate(cases):
        by_p.setdefault(p, []).append(k)
    checked = 0
    for p, ks in by_p.items():
        paths = bm.aligner.align_many([bm.SimilarityMatrix(cases[k][0]) for k in ks], p)
        for k, path in zip(ks, paths):
            S = cases[k][0]
            want = brute_min_cost(S, p)
            assert abs(path.total_cost - want) <= 1e-9
            # the returned path realises the returned cost
            c = sum((1.0 - S[m.i, m.j]) if m.op == "D" else p for m in path.moves)
            assert abs(c - path.total_cost) <= 1e-9
            checked += 1
    assert checked == 625 * 4 + 1000


def _mine_text(pairs, fwd, bwd, lex, cfg) -> str:
    sink = io.StringIO()
    bm.mine_corpus(iter(pairs), fwd, bwd, lex, cfg, sink)
    return sink.getvalue()


def test_05_bidirectional_superset(world500):
    lex, fwd, bwd = world500
    cfg = bm.MinerConfig(bm.MiningParams(0.5, 0.2))
    pairs = list(bm.load_document_pairs(golden("docs40.jsonl")))
    mono = _mine_text(pairs, fwd, None, lex, cfg).count("\n")
    both = _mine_text(pairs, fwd, bwd, lex, cfg).count("\n")
    assert both >= mono > 0

    def const_model(bias, direction):
        return ClassifierModel(schema_id=SCHEMA_ID, weights=[0.0] * 7, bias=bias,
                               direction=direction, default_threshold=0.5,
                               default_penalty=0.2)

    doc = parse_document_pair({"id": "strict", "src_lang": "xx", "tgt_lang": "yy",
                               "src": ["waaa wbbb."], "tgt": ["vaaa vbbb."]}, "mem", 1)
    shy = const_model(-2.0, ("xx", "yy"))   # sigmoid(-2) ~ 0.12 < 0.5
    keen = const_model(+2.0, ("yy", "xx"))  # sigmoid(+2) ~ 0.88 >= 0.5
    assert _mine_text([doc], shy, None, lex, cfg).count("\n") == 0
    assert _mine_text([doc], shy, keen, lex, cfg).count("\n") == 1
