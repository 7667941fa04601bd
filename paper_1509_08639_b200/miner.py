"""End-to-end mining: score, align, filter, merge directions, report.

Same API and output bytes as bimine/miner.py. Where the reference maps
``_mine_task`` over a process pool one document at a time (miner.py:236-245),
this module packs documents into batches and mines a whole batch with one
``bm_mine`` call per model direction; records come back in document order, so
TSV output is written in input order exactly as the reference's ordered
``pool.map`` does. Skip rules (empty side, matrix over MAX_CELLS) and error
propagation points (direction mismatches abort after the preceding documents
were written) are the reference's.
"""

from __future__ import annotations

import json
import logging
import re
import time
from dataclasses import dataclass, field
from typing import IO, Iterable

import numpy as np

from . import aligner
from .aligner import ENGINES, MinedPair, MiningParams
from .classifier import ClassifierModel
from .corpus import DocumentPair, tokenize
from .errors import DataError, ResourceLimitError
from .lexicon import Lexicon

__all__ = [
    "MinedPair",
    "MinerConfig",
    "MiningReport",
    "bidirectional_merge",
    "count_unique_tokens",
    "format_pair_line",
    "mine_corpus",
    "mine_document",
    "mine_documents",
    "report_to_json",
]

log = logging.getLogger(__name__)

# documents packed per bm_mine launch in mine_corpus
BATCH_DOCS = 8192


@dataclass
class MinerConfig:
    params: MiningParams
    workers: int = 1
    engine: str = "sequential"
    wavefront_workers: int = 1
    seed: int = 42

    def __post_init__(self) -> None:
        if self.workers < 1:
            raise ValueError(f"workers {self.workers} must be >= 1")
        if self.wavefront_workers < 1:
            raise ValueError(f"wavefront_workers {self.wavefront_workers} must be >= 1")
        if self.engine not in ENGINES:
            raise ValueError(f"unknown engine {self.engine!r}; choose one of {ENGINES}")


@dataclass
class MiningReport:
    pairs_emitted: int = 0
    unique_src_tokens: int = 0
    unique_tgt_tokens: int = 0
    docs_processed: int = 0
    docs_skipped: int = 0
    wall_clock_seconds: float = 0.0
    per_direction: dict[str, int] = field(default_factory=lambda: {"forward": 0, "backward": 0})


def _orientation(pair: DocumentPair, model: ClassifierModel, lex: Lexicon) -> bool:
    """True when the model reads the pair swapped (miner.py:93-111)."""
    fwd = (pair.source.lang, pair.target.lang)
    bwd = (pair.target.lang, pair.source.lang)
    direction = tuple(model.direction)
    if direction == fwd:
        swapped = False
    elif direction == bwd:
        swapped = True
    else:
        raise DataError(
            f"model direction {direction} matches neither {fwd} nor {bwd} "
            f"for document pair {pair.id!r}"
        )
    if tuple(lex.direction) != direction:
        raise DataError(
            f"lexicon direction {tuple(lex.direction)} does not match model direction {direction}"
        )
    return swapped


def _cap_error(pair: DocumentPair, swapped: bool) -> ResourceLimitError | None:
    n = len(pair.source.sentences)
    m = len(pair.target.sentences)
    if swapped:
        n, m = m, n
    if n * m > aligner.MAX_CELLS:
        return ResourceLimitError(
            f"document pair {pair.id!r} needs a {n}x{m} matrix, over the "
            f"{aligner.MAX_CELLS} cell limit"
        )
    return None


class _Pass:
    """One model direction over a packed batch (lexicon uploaded once)."""

    def __init__(self, dc, corpus, model, lex, cfg):
        from . import engine
        from .pack import pack_lexicon

        self.dc = dc
        self.corpus = corpus
        self.model = model
        self.dl = engine.DeviceLexicon.upload(pack_lexicon(lex, corpus))
        self.cfg = cfg

    def run(self, idx: list[int], swapped: list[bool]):
        from . import engine

        if not idx:
            return np.zeros(0, dtype=np.dtype(engine.N.RECORD_DTYPE))
        view = engine.DocView.of(self.corpus, idx, swapped)
        recs, _cost = engine.mine(self.dc, self.dl, view, self.model,
                                  self.cfg.params.threshold, self.cfg.params.penalty)
        return recs

    def run_device(self, idx: list[int], swapped: list[bool]):
        """The pass's records left on the device: (dense tensor, count)."""
        from . import engine

        view = engine.DocView.of(self.corpus, idx, swapped)
        dense, k, _cost = engine.mine_device(self.dc, self.dl, view, self.model,
                                             self.cfg.params.threshold, self.cfg.params.penalty)
        return dense, k


def _merged_to_pairs(pair: DocumentPair, recs) -> list[MinedPair]:
    """Device-merged records (pair orientation, pad = 1 for backward) ->
    MinedPair objects (miner.py:115-128 labels)."""
    src, tgt = pair.source.sentences, pair.target.sentences
    return [MinedPair(src[i], tgt[j], c, pair.id, "backward" if b else "forward", i, j)
            for i, j, c, b in zip(recs["i"].tolist(), recs["j"].tolist(), recs["conf"].tolist(),
                                  recs["pad"].tolist())]


def _records_to_pairs(pair: DocumentPair, recs, swapped: bool) -> list[MinedPair]:
    src, tgt = pair.source.sentences, pair.target.sentences
    out = []
    for i, j, c in zip(recs["i"].tolist(), recs["j"].tolist(), recs["conf"].tolist()):
        if not swapped:
            out.append(MinedPair(src[i], tgt[j], c, pair.id, "forward", i, j))
        else:  # oriented source is pair.target: re-orient (miner.py:117-128)
            out.append(MinedPair(src[j], tgt[i], c, pair.id, "backward", j, i))
    return out


def _split_by_doc(recs, k: int) -> list:
    if recs.size == 0:
        return [recs] * k
    bounds = np.searchsorted(recs["doc"], np.arange(k + 1))
    return [recs[bounds[q] : bounds[q + 1]] for q in range(k)]


def mine_documents(
    pairs: list[DocumentPair],
    forward: ClassifierModel,
    backward: ClassifierModel | None,
    lex: Lexicon,
    cfg: MinerConfig,
) -> tuple[list[tuple[list[MinedPair], str | None]], Exception | None]:
    """Mine a batch like ``[_mine_task(p) for p in pairs]`` (miner.py:158-180).

    Returns per-document (pairs, skip_reason) for the documents before the
    first one whose task would raise, and that exception (or None).
    """
    from . import engine
    from .pack import Packer

    results: list[tuple[list[MinedPair], str | None] | None] = [None] * len(pairs)
    error: Exception | None = None
    work: list[int] = []
    sw_f: list[bool] = []
    sw_b: list[bool] = []
    rev = lex.reversed() if backward is not None else None
    for k, pair in enumerate(pairs):
        if not pair.source.sentences or not pair.target.sentences:
            side = "src" if not pair.source.sentences else "tgt"
            results[k] = ([], f"document pair {pair.id!r}: empty {side} side")
            continue
        try:
            f = _orientation(pair, forward, lex)
            cap = _cap_error(pair, f)
            if cap is None and backward is not None:
                b = _orientation(pair, backward, rev)
                cap = _cap_error(pair, b)
            else:
                b = False
        except DataError as exc:
            error = exc
            pairs = pairs[:k]
            results = results[:k]
            break
        if cap is not None:
            results[k] = ([], str(cap))
            continue
        work.append(k)
        sw_f.append(f)
        sw_b.append(b)
    if work:
        pk = Packer()
        for k in work:
            pk.add_pair(pairs[k])
        corpus = pk.finish()
        dc = engine.DeviceCorpus.upload(corpus)
        local = list(range(len(work)))
        if backward is None:
            fwd = _split_by_doc(_Pass(dc, corpus, forward, lex, cfg).run(local, sw_f), len(work))
            for q, k in enumerate(work):
                results[k] = (_records_to_pairs(pairs[k], fwd[q], sw_f[q]), None)
        else:
            # both passes stay on the device; bidirectional_merge runs there
            # too (bm_merge_bidir, keyed on the packer's normalized-text ids)
            f, nf = _Pass(dc, corpus, forward, lex, cfg).run_device(local, sw_f)
            b, nb = _Pass(dc, corpus, backward, rev, cfg).run_device(local, sw_b)
            nk = engine.to_dev(corpus.norm_key, engine.device())
            merged = engine.merge_bidir(f, nf, b, nb, corpus.src0, corpus.tgt0, nk, sw_f, sw_b)
            by_doc = _split_by_doc(merged, len(work))
            for q, k in enumerate(work):
                results[k] = (_merged_to_pairs(pairs[k], by_doc[q]), None)
    return [r for r in results if r is not None], error


def mine_document(
    pair: DocumentPair, model: ClassifierModel, lex: Lexicon, cfg: MinerConfig
) -> list[MinedPair]:
    """Mine one document pair with one model (miner.py:84-128)."""
    from . import engine
    from .pack import Packer

    swapped = _orientation(pair, model, lex)
    oriented = DocumentPair(pair.id, pair.target, pair.source) if swapped else pair
    aligner.check_matrix_request(oriented, model)
    pk = Packer()
    pk.add_pair(pair)
    corpus = pk.finish()
    dc = engine.DeviceCorpus.upload(corpus)
    recs = _Pass(dc, corpus, model, lex, cfg).run([0], [swapped])
    return _records_to_pairs(pair, recs, swapped)


def _better(challenger: MinedPair, incumbent: MinedPair) -> bool:
    if challenger.confidence != incumbent.confidence:
        return challenger.confidence > incumbent.confidence
    return challenger.direction == "forward" and incumbent.direction == "backward"


def bidirectional_merge(forward: list[MinedPair], backward: list[MinedPair]) -> list[MinedPair]:
    """Union keyed on normalized text; higher confidence wins, forward wins
    exact ties, first seen otherwise; sorted by (doc, src, tgt) (miner.py:131-155)."""
    best: dict[tuple[str, str], MinedPair] = {}
    for rec in list(forward) + list(backward):
        key = (rec.src.normalized, rec.tgt.normalized)
        cur = best.get(key)
        if cur is None or _better(rec, cur):
            best[key] = rec
    return sorted(best.values(), key=lambda r: (r.doc_id, r.src_index, r.tgt_index))


_FIELD_BREAKS = re.compile(r"[\t\n\r]")


def _sanitize(text: str) -> str:
    return _FIELD_BREAKS.sub(" ", text)


def format_pair_line(rec: MinedPair) -> str:
    return (
        f"{_sanitize(rec.src.raw)}\t{_sanitize(rec.tgt.raw)}\t"
        f"{rec.confidence:.6f}\t{_sanitize(rec.doc_id)}\t{rec.direction}\n"
    )


def mine_corpus(
    doc_pairs: Iterable[DocumentPair],
    forward: ClassifierModel,
    backward: ClassifierModel | None,
    lex: Lexicon,
    cfg: MinerConfig,
    out: IO[str],
) -> MiningReport:
    """Mine a corpus and write TSV records to ``out`` in input order.

    ``cfg.workers`` does not change anything on the GPU path: documents are
    batched (BATCH_DOCS per launch) and output order is input order.
    """
    start = time.perf_counter()
    report = MiningReport()
    if backward is not None:
        lex.reversed()
    src_tokens: set[str] = set()
    tgt_tokens: set[str] = set()
    _mine_stream(doc_pairs, forward, backward, lex, cfg, out, report, src_tokens, tgt_tokens)
    report.unique_src_tokens = len(src_tokens)
    report.unique_tgt_tokens = len(tgt_tokens)
    report.wall_clock_seconds = time.perf_counter() - start
    return report


def _mine_stream(doc_pairs, forward, backward, lex, cfg, out, report: MiningReport,
                 src_tokens: set, tgt_tokens: set) -> None:
    """mine_corpus's body (miner.py:212-245) accumulating into a report and
    token sets (mine_corpus_file resumes here mid-file when a chunk needs the
    Python reader)."""

    def consume(results) -> None:
        for mined, skip_reason in results:
            if skip_reason is not None:
                log.warning("skipping: %s", skip_reason)
                report.docs_skipped += 1
                continue
            report.docs_processed += 1
            for rec in mined:
                out.write(format_pair_line(rec))
                report.pairs_emitted += 1
                report.per_direction[rec.direction] += 1
                src_tokens.update(tokenize(rec.src.normalized))
                tgt_tokens.update(tokenize(rec.tgt.normalized))

    def flush(batch: list[DocumentPair]) -> None:
        results, err = mine_documents(batch, forward, backward, lex, cfg)
        consume(results)
        if err is not None:
            raise err

    if cfg.workers > 1:
        # the reference's pool.map submits every document before the first
        # result is written (miner.py:238-245): a failing iterator writes nothing
        doc_pairs = list(doc_pairs)
    batch: list[DocumentPair] = []
    it = iter(doc_pairs)
    while True:
        try:
            pair = next(it)
        except StopIteration:
            break
        except BaseException:
            # workers=1 maps lazily (miner.py:236-237): every document read
            # before the failing one is mined and written (or its own task
            # error wins), then the iterator's exception propagates
            if batch:
                flush(batch)
            raise
        batch.append(pair)
        if len(batch) >= BATCH_DOCS:
            flush(batch)
            batch = []
    if batch:
        flush(batch)


def count_unique_tokens(pairs: list[MinedPair]) -> tuple[int, int]:
    src_tokens: set[str] = set()
    tgt_tokens: set[str] = set()
    for rec in pairs:
        src_tokens.update(tokenize(rec.src.normalized))
        tgt_tokens.update(tokenize(rec.tgt.normalized))
    return (len(src_tokens), len(tgt_tokens))


def report_to_json(report: MiningReport) -> str:
    payload = {
        "pairs_emitted": report.pairs_emitted,
        "unique_src_tokens": report.unique_src_tokens,
        "unique_tgt_tokens": report.unique_tgt_tokens,
        "docs_processed": report.docs_processed,
        "docs_skipped": report.docs_skipped,
        "wall_clock_seconds": report.wall_clock_seconds,
        "per_direction": dict(report.per_direction),
    }
    return json.dumps(payload, sort_keys=True, indent=2) + "\n"
