"""Host packing: DocumentPair objects -> the flat id arrays of bm_sentences /
bm_docs / bm_lexicon (include/bimine_b200.h), and their device upload.

Per sentence the scoring kernel needs exactly what extract_features reads
(bimine/classifier.py:54-97, lexicon.py:95-105), taken from ``Sentence.tokens``:

* T = len(tokens), P = #tokens without an alphanumeric character,
* |A| = #tokens with ``str.isalpha()``,
* U = {normalize(t)} as interned ids (ascending), each with the number of
  isalpha() tokens that normalize to it (A as a multiset),
* D = {t : t.isdigit()} (raw strings) as interned ids.

The lexicon is lowered to CSR over the same id space: a candidate string that
occurs nowhere in the batch can never be "in the target token set", so it is
dropped. The reverse table is the caller's ``lex.reversed()`` itself.
"""

from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np

from .corpus import DocumentPair, Sentence, normalize



@dataclass
class PackedCorpus:
    n_tok: np.ndarray
    n_punct: np.ndarray
    n_alpha: np.ndarray
    tok_off: np.ndarray
    tok_id: np.ndarray
    tok_alpha: np.ndarray
    dig_off: np.ndarray
    dig_id: np.ndarray
    src0: np.ndarray
    n: np.ndarray
    tgt0: np.ndarray
    m: np.ndarray
    strings: list[str] = field(default_factory=list)
    ids: dict[str, int] = field(default_factory=dict)
    # per sentence: an id of its normalized text (bidirectional_merge's key)
    norm_key: np.ndarray | None = None

    @property
    def n_sent(self) -> int:
        return int(self.n_tok.shape[0])

    @property
    def n_docs(self) -> int:
        return int(self.n.shape[0])

    def doc_token_max(self) -> np.ndarray:
        """Largest token count T of any sentence of each doc (routing input of
        bm_mine: T bounds |A|, P and |D|, so T <= 255 lets the fused kernel
        keep all four in one byte each)."""
        out = np.zeros(self.n_docs, dtype=np.int32)
        if self.n_sent == 0 or self.n_docs == 0:
            return out
        a = np.append(self.n_tok, 0).astype(np.int32)  # sentinel: e may equal n_sent
        for lo, cnt in ((self.src0, self.n), (self.tgt0, self.m)):
            lo = lo.astype(np.int64)
            ind = np.empty(2 * lo.size, dtype=np.int64)
            ind[0::2] = lo
            ind[1::2] = lo + cnt
            seg = np.maximum.reduceat(a, ind)[0::2]
            out = np.maximum(out, np.where(cnt > 0, seg, 0))
        return out.astype(np.int32)

    def swapped(self) -> "PackedCorpus":
        """Same sentences with source and target sides exchanged (the backward
        model's orientation, miner.py:99-101): only the doc table changes."""
        return PackedCorpus(self.n_tok, self.n_punct, self.n_alpha, self.tok_off, self.tok_id,
                            self.tok_alpha, self.dig_off, self.dig_id, self.tgt0, self.m,
                            self.src0, self.n, self.strings, self.ids)


class Packer:
    """Interns token strings and appends sentences / document pairs."""

    def __init__(self) -> None:
        self.ids: dict[str, int] = {}
        self.strings: list[str] = []
        self._tok: dict[str, tuple[int, bool, int, bool]] = {}
        self._T: list[int] = []
        self._P: list[int] = []
        self._A: list[int] = []
        self._tok_off: list[int] = [0]
        self._tok_id: list[int] = []
        self._tok_alpha: list[int] = []
        self._dig_off: list[int] = [0]
        self._dig_id: list[int] = []
        self._docs: list[tuple[int, int, int, int]] = []
        self._norm: dict[str, int] = {}
        self._norm_key: list[int] = []

    def intern(self, s: str) -> int:
        k = self.ids.get(s)
        if k is None:
            k = len(self.strings)
            self.ids[s] = k
            self.strings.append(s)
        return k

    def _token(self, t: str) -> tuple[int, bool, int, bool]:
        info = self._tok.get(t)
        if info is None:
            nid = self.intern(normalize(t))
            did = self.intern(t) if t.isdigit() else -1
            punct = not any(c.isalnum() for c in t)
            info = (nid, t.isalpha(), did, punct)
            self._tok[t] = info
        return info

    def add_sentence(self, sent: Sentence) -> int:
        alpha: dict[int, int] = {}
        digits: set[int] = set()
        punct = 0
        n_alpha = 0
        for t in sent.tokens:
            nid, is_alpha, did, is_punct = self._token(t)
            if is_alpha:
                alpha[nid] = alpha.get(nid, 0) + 1
                n_alpha += 1
            elif nid not in alpha:
                alpha[nid] = 0
            if did >= 0:
                digits.add(did)
            punct += is_punct
        idx = len(self._T)
        self._norm_key.append(self._norm.setdefault(sent.normalized, len(self._norm)))
        self._T.append(len(sent.tokens))
        self._P.append(punct)
        self._A.append(n_alpha)
        for nid in sorted(alpha):
            self._tok_id.append(nid)
            self._tok_alpha.append(alpha[nid])
        self._tok_off.append(len(self._tok_id))
        self._dig_id.extend(sorted(digits))
        self._dig_off.append(len(self._dig_id))
        return idx

    def add_pair(self, pair: DocumentPair) -> int:
        src0 = len(self._T)
        for s in pair.source.sentences:
            self.add_sentence(s)
        tgt0 = len(self._T)
        for s in pair.target.sentences:
            self.add_sentence(s)
        self._docs.append((src0, len(pair.source.sentences), tgt0, len(pair.target.sentences)))
        return len(self._docs) - 1

    def add_sentence_pair(self, src: Sentence, tgt: Sentence) -> tuple[int, int]:
        return self.add_sentence(src), self.add_sentence(tgt)

    def finish(self) -> PackedCorpus:
        d = np.asarray(self._docs, dtype=np.int32).reshape(-1, 4)
        return PackedCorpus(
            n_tok=np.asarray(self._T, dtype=np.int32),
            n_punct=np.asarray(self._P, dtype=np.int32),
            n_alpha=np.asarray(self._A, dtype=np.int32),
            tok_off=np.asarray(self._tok_off, dtype=np.int32),
            tok_id=np.asarray(self._tok_id, dtype=np.int32),
            tok_alpha=np.asarray(self._tok_alpha, dtype=np.uint32),
            dig_off=np.asarray(self._dig_off, dtype=np.int32),
            dig_id=np.asarray(self._dig_id, dtype=np.int32),
            src0=np.ascontiguousarray(d[:, 0]),
            n=np.ascontiguousarray(d[:, 1]),
            tgt0=np.ascontiguousarray(d[:, 2]),
            m=np.ascontiguousarray(d[:, 3]),
            strings=self.strings,
            ids=self.ids,
            norm_key=np.asarray(self._norm_key, dtype=np.int32),
        )


def pack_pairs(pairs: list[DocumentPair]) -> PackedCorpus:
    pk = Packer()
    for p in pairs:
        pk.add_pair(p)
    return pk.finish()


@dataclass
class PackedLexicon:
    n_ids: int
    fwd_off: np.ndarray
    fwd_cand: np.ndarray
    rev_off: np.ndarray
    rev_cand: np.ndarray

    def swapped(self) -> "PackedLexicon":
        return PackedLexicon(self.n_ids, self.rev_off, self.rev_cand, self.fwd_off, self.fwd_cand)


def _csr(entries: dict, strings: list[str], ids: dict[str, int]) -> tuple[np.ndarray, np.ndarray]:
    off = np.zeros(len(strings) + 1, dtype=np.int32)
    cand: list[int] = []
    for k, s in enumerate(strings):
        got = entries.get(s)
        if got:
            present = sorted({ids[c] for c, _p in got if c in ids})
            cand.extend(present)
        off[k + 1] = len(cand)
    return off, np.asarray(cand, dtype=np.int32)


def pack_lexicon(lex, corpus: PackedCorpus) -> PackedLexicon:
    """Forward CSR from ``lex.entries`` and reverse CSR from ``lex.reversed()``
    (coverage looks words up with ``entries.get``, lexicon.py:103)."""
    fo, fc = _csr(lex.entries, corpus.strings, corpus.ids)
    ro, rc = _csr(lex.reversed().entries, corpus.strings, corpus.ids)
    return PackedLexicon(len(corpus.strings), fo, fc, ro, rc)
