"""Synthetic comparable corpora in the shape of the reference's generator.

The reference's test generator (pkg/tests/synthgen.py:19-145) builds paired
vocabularies ``w<abc>`` <-> ``v<abc>``, a one-to-one lexicon with probability
0.9, word-for-word translation pairs of 4-9 words (+ a 4-digit year with
probability 0.15, target words noised with probability ``noise``) and
one-sided distractors, each ending in ".". This module draws the same
distributions with numpy and emits the packed id arrays directly (the
benchmark corpora have up to ~10^8 sentences, far beyond what a per-sentence
Python generator can produce), and can render any subset as text
``DocumentPair`` objects so tests can round-trip it through the real packer.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from .corpus import Document, DocumentPair, Sentence
from .lexicon import Lexicon
from .pack import PackedCorpus, PackedLexicon

SRC_LANG, TGT_LANG = "xx", "yy"
YEAR0, NYEARS = 1900, 131


def letters(k: int) -> str:
    out = []
    for _ in range(3):
        out.append(chr(ord("a") + k % 26))
        k //= 26
    return "".join(reversed(out))


@dataclass
class SynthWorld:
    """Id layout: src word k -> k, tgt word k -> V+k, "." -> 2V, years after."""

    vocab: int

    @property
    def dot(self) -> int:
        return 2 * self.vocab

    def year_id(self, y):
        return 2 * self.vocab + 1 + (np.asarray(y) - YEAR0)

    @property
    def n_ids(self) -> int:
        return 2 * self.vocab + 1 + NYEARS

    def strings(self) -> list[str]:
        V = self.vocab
        return ([f"w{letters(k)}" for k in range(V)] + [f"v{letters(k)}" for k in range(V)]
                + ["."] + [str(YEAR0 + y) for y in range(NYEARS)])

    def lexicon(self) -> Lexicon:
        return Lexicon(direction=(SRC_LANG, TGT_LANG),
                       entries={f"w{letters(k)}": [(f"v{letters(k)}", 0.9)] for k in range(self.vocab)})

    def packed_lexicon(self) -> PackedLexicon:
        V, n = self.vocab, self.n_ids
        fwd_off = np.zeros(n + 1, dtype=np.int32)
        fwd_off[1 : V + 1] = np.arange(1, V + 1)
        fwd_off[V + 1 :] = V
        rev_off = np.zeros(n + 1, dtype=np.int32)
        rev_off[V + 1 : 2 * V + 1] = np.arange(1, V + 1)
        rev_off[2 * V + 1 :] = V
        return PackedLexicon(n, fwd_off, np.arange(V, 2 * V, dtype=np.int32), rev_off,
                             np.arange(V, dtype=np.int32))


@dataclass
class SynthCorpus:
    world: SynthWorld
    packed: PackedCorpus
    # per sentence token lists (for text rendering): flat ids + offsets
    tok_flat: np.ndarray
    tok_start: np.ndarray
    gold: list[np.ndarray]  # per doc: (k, 2) gold (i, j)

    def doc_pairs(self, idx) -> list[DocumentPair]:
        strings = self.world.strings()
        c = self.packed
        out = []
        for d in idx:
            def side(s0, cnt):
                sents = []
                for s in range(s0, s0 + cnt):
                    ids = self.tok_flat[self.tok_start[s] : self.tok_start[s + 1]]
                    words = [strings[t] for t in ids if t != self.world.dot]
                    sents.append(Sentence.from_text(" ".join(words) + "."))
                return sents
            src = side(int(c.src0[d]), int(c.n[d]))
            tgt = side(int(c.tgt0[d]), int(c.m[d]))
            out.append(DocumentPair(f"doc{d:07d}", Document(f"doc{d:07d}", SRC_LANG, src),
                                    Document(f"doc{d:07d}", TGT_LANG, tgt)))
        return out


def make_corpus(n_gold, n_src, n_tgt, vocab: int = 5000, noise: float = 0.1, seed: int = 0,
                digit_rate: float = 0.15) -> SynthCorpus:
    """Docs d with n_gold[d] translation pairs and n_src[d] / n_tgt[d]
    distractors, events shuffled (synthgen.make_comparable_doc)."""
    rng = np.random.default_rng(seed)
    W = SynthWorld(vocab)
    V = vocab
    g = np.asarray(n_gold, dtype=np.int64)
    a = np.asarray(n_src, dtype=np.int64)
    b = np.asarray(n_tgt, dtype=np.int64)
    D = g.size
    ev_n = g + a + b
    E = int(ev_n.sum())
    ev_doc = np.repeat(np.arange(D), ev_n)
    ev_type = np.concatenate([np.repeat([0, 1, 2], [gg, aa, bb]) for gg, aa, bb in zip(g, a, b)]) \
        if D < 2000 else _types_fast(g, a, b)
    # shuffle events within each doc
    order = np.lexsort((rng.random(E), ev_doc))
    ev_type = ev_type[order]
    # sentences: per doc, source side = events of type 0/1 in order, then target = 0/2
    is_src = ev_type != 2
    is_tgt = ev_type != 1
    n = np.bincount(ev_doc[is_src], minlength=D)
    m = np.bincount(ev_doc[is_tgt], minlength=D)
    # ordinal of each event within its side
    src_rank = _rank_within(ev_doc, is_src)
    tgt_rank = _rank_within(ev_doc, is_tgt)
    doc_base = np.zeros(D, dtype=np.int64)
    doc_base[1:] = np.cumsum(n + m)[:-1]
    src0 = doc_base
    tgt0 = doc_base + n
    S = int((n + m).sum())

    # words: each event gets k in [4, 9] words
    k = rng.integers(4, 10, size=E)
    kmax = 9
    words = rng.integers(0, V, size=(E, kmax))
    # gold pairs use distinct words: redraw duplicates
    gold_ev = ev_type == 0
    pos = np.arange(kmax)[None, :]
    valid = pos < k[:, None]
    for _ in range(32):
        s2 = np.sort(np.where(valid, words, -1 - pos), axis=1)
        bad = gold_ev & (s2[:, 1:] == s2[:, :-1]).any(axis=1)
        if not bad.any():
            break
        words[bad] = rng.integers(0, V, size=(int(bad.sum()), kmax))
    year = np.where(rng.random(E) < digit_rate, rng.integers(YEAR0, YEAR0 + NYEARS, size=E), -1)
    noise_mask = rng.random((E, kmax)) < noise
    noise_words = rng.integers(0, V, size=(E, kmax))

    # source sentence of event e (types 0, 1): words are src ids; type-2 events have none
    src_words = words
    tgt_words = np.where(ev_type[:, None] == 0, np.where(noise_mask, noise_words, words), words) + V
    sent_src = np.where(is_src, src0[ev_doc] + src_rank, -1)
    sent_tgt = np.where(is_tgt, tgt0[ev_doc] + tgt_rank, -1)
    has_year_src = (year >= 0) & (ev_type == 0)
    has_year_tgt = has_year_src

    tok_sent = []
    tok_id = []
    tok_alpha = []
    for sel, sent, wmat, hy in ((is_src, sent_src, src_words, has_year_src),
                               (is_tgt, sent_tgt, tgt_words, has_year_tgt)):
        ev = np.nonzero(sel)[0]
        vv = valid[ev]
        ss = np.repeat(sent[ev], vv.sum(axis=1))
        tok_sent.append(ss)
        tok_id.append(wmat[ev][vv])
        tok_alpha.append(np.ones(ss.size, dtype=np.int64))
        ey = ev[hy[ev]]
        tok_sent.append(sent[ey])
        tok_id.append(W.year_id(year[ey]))
        tok_alpha.append(np.zeros(ey.size, dtype=np.int64))
        tok_sent.append(sent[ev])
        tok_id.append(np.full(ev.size, W.dot))
        tok_alpha.append(np.zeros(ev.size, dtype=np.int64))
    ts = np.concatenate(tok_sent)
    ti = np.concatenate(tok_id).astype(np.int64)
    ta = np.concatenate(tok_alpha)
    # raw token lists in sentence order (for text rendering): words, then year, then "."
    o = np.argsort(ts, kind="stable")
    tok_flat = ti[o].astype(np.int32)
    tok_start = np.zeros(S + 1, dtype=np.int64)
    np.cumsum(np.bincount(ts, minlength=S), out=tok_start[1:])
    T = np.bincount(ts, minlength=S).astype(np.int32)
    nA = np.bincount(ts, weights=ta, minlength=S).astype(np.int32)
    P = np.bincount(ts[ti == W.dot], minlength=S).astype(np.int32)
    # unique (sentence, id) with alpha multiplicities
    key = ts * W.n_ids + ti
    uk, inv = np.unique(key, return_inverse=True)
    alpha = np.bincount(inv, weights=ta, minlength=uk.size).astype(np.uint32)
    u_sent = uk // W.n_ids
    u_id = (uk % W.n_ids).astype(np.int32)
    tok_off = np.zeros(S + 1, dtype=np.int32)
    np.cumsum(np.bincount(u_sent, minlength=S), out=tok_off[1:])
    dig = (u_id > W.dot)
    dig_sent = u_sent[dig]
    dig_off = np.zeros(S + 1, dtype=np.int32)
    np.cumsum(np.bincount(dig_sent, minlength=S), out=dig_off[1:])
    packed = PackedCorpus(
        n_tok=T, n_punct=P, n_alpha=nA, tok_off=tok_off, tok_id=u_id, tok_alpha=alpha,
        dig_off=dig_off, dig_id=u_id[dig].astype(np.int32),
        src0=src0.astype(np.int32), n=n.astype(np.int32), tgt0=tgt0.astype(np.int32),
        m=m.astype(np.int32),
    )
    # gold cells per doc
    ge = np.nonzero(gold_ev)[0]
    gi, gj, gd = src_rank[ge], tgt_rank[ge], ev_doc[ge]
    bounds = np.searchsorted(gd, np.arange(D + 1))
    gold = [np.stack([gi[bounds[d]:bounds[d + 1]], gj[bounds[d]:bounds[d + 1]]], axis=1)
            for d in range(D)] if D <= 200000 else []
    return SynthCorpus(W, packed, tok_flat, tok_start, gold)


def _types_fast(g, a, b) -> np.ndarray:
    n = g + a + b
    D = n.size
    start = np.zeros(D, dtype=np.int64)
    start[1:] = np.cumsum(n)[:-1]
    E = int(n.sum())
    idx = np.arange(E) - np.repeat(start, n)
    gg = np.repeat(g, n)
    aa = np.repeat(a, n)
    return np.where(idx < gg, 0, np.where(idx < gg + aa, 1, 2))


def _rank_within(doc: np.ndarray, sel: np.ndarray) -> np.ndarray:
    """0-based rank of each selected event among the selected events of its doc."""
    c = np.cumsum(sel) - sel
    first = np.zeros(doc.size, dtype=np.int64)
    starts = np.nonzero(np.r_[True, doc[1:] != doc[:-1]])[0]
    base = c[starts]
    first = np.repeat(base, np.diff(np.r_[starts, doc.size]))
    return np.where(sel, c - first, -1)


def c2_shape(n_docs: int = 10000):
    """BASELINE config 2: ~100 x 100 (60 gold + 40/40 distractors)."""
    return (np.full(n_docs, 60), np.full(n_docs, 40), np.full(n_docs, 40))


def c3_shape(n_docs: int, seed: int = 2026):
    """BASELINE config 3: skewed lengths, n = clip(LogNormal(ln 60, 1), 10, 2000),
    m = clip(n * LogNormal(0, 0.25), 10, 2000), ~60% of min(n, m) gold."""
    r = np.random.default_rng(seed)
    n = np.clip(np.rint(np.exp(r.normal(np.log(60), 1.0, n_docs))), 10, 2000).astype(np.int64)
    m = np.clip(np.rint(n * np.exp(r.normal(0.0, 0.25, n_docs))), 10, 2000).astype(np.int64)
    g = np.floor(0.6 * np.minimum(n, m)).astype(np.int64)
    return g, n - g, m - g


class _SynthHandle:
    """Owns a bm_synth corpus; numpy views of its arrays keep it alive."""

    def __init__(self, lib, h):
        self.lib, self.h = lib, h

    def __del__(self):
        if self.h:
            self.lib.bm_synth_free(self.h)
            self.h = None


def _view(owner, ptr: int, count: int, dtype) -> np.ndarray:
    import ctypes as C

    dt = np.dtype(dtype)
    if count == 0:
        return np.zeros(0, dtype=dt)
    buf = (C.c_char * (count * dt.itemsize)).from_address(ptr)
    a = np.frombuffer(buf, dtype=dt, count=count)
    a.flags.writeable = False
    # the view's base chain ends in `buf`; hang the owner on it
    buf._owner = owner
    return a


@dataclass
class NativeSynthCorpus:
    """Output of make_corpus_native: the packed batch plus per-doc gold cells
    (gold_off[d] .. gold_off[d+1] into gold_i / gold_j)."""

    world: SynthWorld
    packed: PackedCorpus
    gold_off: np.ndarray
    gold_i: np.ndarray
    gold_j: np.ndarray

    def gold_keys(self) -> list[np.ndarray]:
        """Per-doc gold keys i * m + j (ascending), the tuner's device layout."""
        m = self.packed.m.astype(np.int64)
        key = self.gold_i.astype(np.int64) * np.repeat(m, np.diff(self.gold_off)) + self.gold_j
        return [np.sort(key[self.gold_off[d]:self.gold_off[d + 1]]) for d in range(len(m))]


def make_corpus_native(n_gold, n_src, n_tgt, ids=None, vocab: int = 5000, noise: float = 0.1,
                       seed: int = 0, digit_rate: float = 0.15, threads: int = 0
                       ) -> NativeSynthCorpus:
    """make_corpus's distributions, generated natively (csrc/bm_synth.cpp) per
    document from a stream keyed by (seed, ids[q]): a shard of a corpus is
    generated on its own and holds the same documents as the whole corpus."""
    import ctypes as C

    from . import _native as N

    lib = N.load_library()
    g = np.ascontiguousarray(n_gold, dtype=np.int32)
    a = np.ascontiguousarray(n_src, dtype=np.int32)
    b = np.ascontiguousarray(n_tgt, dtype=np.int32)
    k = g.size
    ids = np.arange(k, dtype=np.int64) if ids is None else np.ascontiguousarray(ids, np.int64)
    spec = N.SynthSpec(int(vocab), float(noise), float(digit_rate), int(seed) & (2**64 - 1))
    h = C.c_void_p()
    rc = lib.bm_synth_generate(C.byref(spec), ids.ctypes.data, g.ctypes.data, a.ctypes.data,
                               b.ctypes.data, k, int(threads), C.byref(h))
    if rc != 0:
        raise ValueError(f"bm_synth_generate failed ({rc})")
    owner = _SynthHandle(lib, h.value)
    v = N.SynthArrays()
    lib.bm_synth_view(h, C.byref(v))
    S, E, G, D = v.n_sent, v.n_tok_entries, v.n_dig_entries, v.n_docs
    i32 = np.int32
    packed = PackedCorpus(
        n_tok=_view(owner, v.n_tok, S, i32), n_punct=_view(owner, v.n_punct, S, i32),
        n_alpha=_view(owner, v.n_alpha, S, i32), tok_off=_view(owner, v.tok_off, S + 1, i32),
        tok_id=_view(owner, v.tok_id, E, i32), tok_alpha=_view(owner, v.tok_alpha, E, np.uint32),
        dig_off=_view(owner, v.dig_off, S + 1, i32), dig_id=_view(owner, v.dig_id, G, i32),
        src0=_view(owner, v.src0, D, i32), n=_view(owner, v.n, D, i32),
        tgt0=_view(owner, v.tgt0, D, i32), m=_view(owner, v.m, D, i32),
    )
    return NativeSynthCorpus(SynthWorld(vocab), packed, _view(owner, v.gold_off, D + 1, np.int64),
                             _view(owner, v.gold_i, v.n_gold, i32),
                             _view(owner, v.gold_j, v.n_gold, i32))


def write_jsonl_native(path: str, n_gold, n_src, n_tgt, ids=None, vocab: int = 5000,
                       noise: float = 0.1, seed: int = 0, digit_rate: float = 0.15,
                       threads: int = 0) -> None:
    """make_corpus_native's documents as document-pair JSONL text (the words,
    then the year, then "."; ids "doc%07d" of the global document index)."""
    import ctypes as C

    from . import _native as N

    lib = N.load_library()
    g = np.ascontiguousarray(n_gold, dtype=np.int32)
    a = np.ascontiguousarray(n_src, dtype=np.int32)
    b = np.ascontiguousarray(n_tgt, dtype=np.int32)
    ids = np.arange(g.size, dtype=np.int64) if ids is None else np.ascontiguousarray(ids, np.int64)
    spec = N.SynthSpec(int(vocab), float(noise), float(digit_rate), int(seed) & (2**64 - 1))
    rc = lib.bm_synth_jsonl(C.byref(spec), ids.ctypes.data, g.ctypes.data, a.ctypes.data,
                            b.ctypes.data, g.size, int(threads), path.encode())
    if rc != 0:
        raise OSError(f"bm_synth_jsonl failed ({rc})")
