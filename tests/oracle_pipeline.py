"""Test helper: the reference mining pipeline driven by the CPU oracle.

Reuses the package's host-side pieces (packing, orientation rules, merge,
TSV formatting) and replaces every GPU call with the oracle, so a test can
compare "GPU path" and "oracle path" outputs byte for byte, and pin the
oracle path itself against the reference's golden TSVs.
"""

from __future__ import annotations

import io

import numpy as np

import paper_1509_08639_b200 as bm
from paper_1509_08639_b200 import miner
from paper_1509_08639_b200.pack import pack_lexicon, pack_pairs


def oracle_records(oracle, pairs, model, lex, swapped, t, p, threads=4):
    corpus = pack_pairs(pairs)
    plex = pack_lexicon(lex, corpus)
    sw = np.asarray(swapped, dtype=bool)
    s0 = np.where(sw, corpus.tgt0, corpus.src0)
    t0 = np.where(sw, corpus.src0, corpus.tgt0)
    n = np.where(sw, corpus.m, corpus.n)
    m = np.where(sw, corpus.n, corpus.m)
    hb = oracle.HostBatch(corpus, plex, s0, n, t0, m)
    recs, cost = oracle.mine(hb, model, t, p, threads=threads)
    return recs, cost


def oracle_mine_text(oracle, pairs, fwd, bwd, lex, t=0.5, p=0.2):
    """mine_corpus (miner.py:197-250) with the oracle as the compute engine."""
    out = io.StringIO()
    sf = [miner._orientation(x, fwd, lex) for x in pairs]
    rf, _ = oracle_records(oracle, pairs, fwd, lex, sf, t, p)
    by_doc_f = miner._split_by_doc(rf, len(pairs))
    if bwd is not None:
        rev = lex.reversed()
        sb = [miner._orientation(x, bwd, rev) for x in pairs]
        rb, _ = oracle_records(oracle, pairs, bwd, rev, sb, t, p)
        by_doc_b = miner._split_by_doc(rb, len(pairs))
    for k, pair in enumerate(pairs):
        mined = miner._records_to_pairs(pair, by_doc_f[k], sf[k])
        if bwd is not None:
            mined = bm.bidirectional_merge(mined, miner._records_to_pairs(pair, by_doc_b[k], sb[k]))
        for rec in mined:
            out.write(bm.format_pair_line(rec))
    return out.getvalue()


def oracle_tune_trace(oracle, model, lex, dev, thresholds, penalties):
    corpus = pack_pairs(dev.docs)
    hb = oracle.HostBatch(corpus, pack_lexicon(lex, corpus))
    uniq_p = sorted(set(float(x) for x in penalties))
    uniq_t = sorted(set(float(x) for x in thresholds))
    gold = [np.asarray(sorted(i * int(corpus.m[q]) + j for i, j in dev.gold[q]), np.int64)
            for q in range(len(dev.docs))]
    pred, hit = oracle.tune(hb, model, uniq_p, uniq_t, gold, threads=4)
    n_gold = sum(len(g) for g in dev.gold)
    trace = []
    for t in thresholds:
        for p in penalties:
            a, b = uniq_p.index(float(p)), uniq_t.index(float(t))
            trace.append((t, p) + bm.tuner._prf(int(pred[a, b]), n_gold, int(hit[a, b])))
    return trace
