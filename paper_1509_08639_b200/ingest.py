"""Native corpus path behind the reference's API.

``mine_corpus_file(path, forward, backward, lex, cfg, out)`` produces exactly
what ``mine_corpus(load_document_pairs(path), forward, backward, lex, cfg,
out)`` produces -- the same TSV bytes and the same ``MiningReport`` counts --
but reads, segments, tokenizes and packs the JSONL file in C++
(``csrc/bm_ingest.cpp``), lowers the lexicon there, mines on the GPU, and
merges / formats the records in C++ too.

The native reader accepts a file only when it can reproduce Python's Unicode
semantics exactly (valid UTF-8, JSON inside a validated subset, string or
integer ids, text that NFC leaves unchanged and that lowercases character by
character -- see the contract at the top of bm_ingest.cpp); anything else -- and any document whose orientation check would
raise -- takes the Python path, which is the reference behaviour by
construction. Empty-side pairs are reported through ``on_skip`` (and the log)
before mining starts rather than interleaved with the output; the TSV and the
report do not depend on that order.
"""

from __future__ import annotations

import ctypes as C
import logging
import time
from typing import IO, Callable

import numpy as np

from . import _native as N
from .classifier import ClassifierModel
from .lexicon import Lexicon
from .pack import PackedCorpus, PackedLexicon

log = logging.getLogger(__name__)

# phase timings (seconds) of the last mine_corpus_file call on the native path
LAST_TIMINGS: dict[str, float] = {}

_SENT_FIELDS = (("n_tok", np.int32, "n_sent"), ("n_punct", np.int32, "n_sent"),
                ("n_alpha", np.int32, "n_sent"), ("tok_off", np.int32, "n_sent+1"),
                ("tok_id", np.int32, "n_tok_entries"), ("tok_alpha", np.uint32, "n_tok_entries"),
                ("dig_off", np.int32, "n_sent+1"), ("dig_id", np.int32, "n_dig_entries"),
                ("src0", np.int32, "n_docs"), ("n", np.int32, "n_docs"),
                ("tgt0", np.int32, "n_docs"), ("m", np.int32, "n_docs"))


def _bytes_at(ptr, n: int) -> bytes:
    """n bytes at ptr (ctypes.string_at takes a C int size: it truncates
    lengths of 2 GiB and more, e.g. the TSV of a whole C3 corpus)."""
    if n <= 0:
        return b""
    addr = ptr.value if isinstance(ptr, (C.c_char_p, C.c_void_p)) else ptr
    if isinstance(ptr, C.c_char_p):
        addr = C.cast(ptr, C.c_void_p).value
    return bytes((C.c_char * n).from_address(addr))


def _view(ptr: int, dtype, count: int) -> np.ndarray:
    if count == 0 or not ptr:
        return np.zeros(0, dtype=dtype)
    buf = (C.c_char * (count * np.dtype(dtype).itemsize)).from_address(ptr)
    return np.frombuffer(buf, dtype=dtype, count=count)


class NativeCorpus:
    """A JSONL file ingested by bm_ingest_jsonl (arrays owned by the handle)."""

    def __init__(self, handle: int):
        self._lib = N.load_library()
        self._h = C.c_void_p(handle)
        a = N.IngestArrays()
        N.check(self._lib.bm_ingest_view(self._h, C.byref(a)))
        sizes = {"n_sent": a.n_sent, "n_sent+1": a.n_sent + 1, "n_docs": a.n_docs,
                 "n_tok_entries": a.n_tok_entries, "n_dig_entries": a.n_dig_entries}
        arrs = {name: _view(getattr(a, name), dt, sizes[sz]) for name, dt, sz in _SENT_FIELDS}
        self.n_ids = a.n_ids
        self.packed = PackedCorpus(**arrs)
        self.doc_ids: list[str] = []
        self.langs: list[tuple[str, str]] = []
        pid, psl, ptl = C.c_char_p(), C.c_char_p(), C.c_char_p()
        for k in range(a.n_docs):
            N.check(self._lib.bm_ingest_doc(self._h, k, C.byref(pid), C.byref(psl), C.byref(ptl)))
            self.doc_ids.append(pid.value.decode("utf-8"))
            self.langs.append((psl.value.decode("utf-8"), ptl.value.decode("utf-8")))
        self.skipped: list[tuple[int, str, str]] = []
        ln = C.c_int64()
        for q in range(a.n_skipped):
            N.check(self._lib.bm_ingest_skipped(self._h, q, C.byref(ln), C.byref(pid), C.byref(psl)))
            self.skipped.append((ln.value, pid.value.decode("utf-8"), psl.value.decode("utf-8")))

    @classmethod
    def load_range(cls, path: str, b0: int, b1: int, line0: int) -> "NativeCorpus | None":
        """Ingest the lines of bytes [b0, b1) (numbered from line0 + 1); None
        when they are outside the native subset."""
        lib = N.load_library()
        h = C.c_void_p()
        nl = C.c_int64()
        why = C.create_string_buffer(256)
        rc = lib.bm_ingest_jsonl_range(path.encode(), int(b0), int(b1), int(line0), C.byref(h),
                                       C.byref(nl), why, len(why))
        if rc == N.BM_EUNSUPPORTED:
            log.info("native ingest declined %s bytes [%d, %d) (%s); using the Python reader",
                     path, b0, b1, why.value.decode("ascii", "replace"))
            return None
        N.check(rc)
        out = cls(h.value)
        out.n_lines = nl.value
        return out

    @classmethod
    def load(cls, path: str, gold: bool = False) -> "NativeCorpus | None":
        """Ingest ``path`` (a gold set when ``gold``); None when it is outside
        the native subset or would make the Python reader raise."""
        lib = N.load_library()
        h = C.c_void_p()
        why = C.create_string_buffer(256)
        fn = lib.bm_ingest_gold_jsonl if gold else lib.bm_ingest_jsonl
        rc = fn(path.encode(), C.byref(h), why, len(why))
        if rc == N.BM_EUNSUPPORTED:
            log.info("native ingest declined %s (%s); using the Python reader", path,
                     why.value.decode("ascii", "replace"))
            return None
        N.check(rc)
        out = cls(h.value)
        if gold:
            keys, off, nk = C.c_void_p(), C.c_void_p(), C.c_int64()
            N.check(lib.bm_ingest_gold(out._h, C.byref(keys), C.byref(off), C.byref(nk)))
            out.gold_off = _view(off.value, np.int64, out.packed.n_docs + 1)
            out.gold_keys = _view(keys.value, np.int64, nk.value)
        return out

    def __del__(self):
        h = getattr(self, "_h", None)
        if h is not None and h.value:
            self._lib.bm_ingest_free(h)
            self._h = None

    def lexicon(self, lex: Lexicon) -> PackedLexicon:
        """pack_lexicon(lex, corpus) computed natively (forward entries; the
        reverse CSR is their transpose, i.e. lex.reversed())."""
        src: list[bytes] = []
        tgt: list[bytes] = []
        for word, cands in lex.entries.items():
            wb = word.encode("utf-8")
            for c, _p in cands:
                src.append(wb)
                tgt.append(c.encode("utf-8"))
        n = len(src)
        sa = (C.c_char_p * max(n, 1))(*src)
        ta = (C.c_char_p * max(n, 1))(*tgt)
        out = N.LexiconC()
        N.check(self._lib.bm_ingest_lexicon(self._h, sa, ta, n, C.byref(out)))
        nid = self.n_ids
        nf = int(_view(out.fwd_off, np.int32, nid + 1)[-1]) if nid else 0
        nr = int(_view(out.rev_off, np.int32, nid + 1)[-1]) if nid else 0
        return PackedLexicon(nid, _view(out.fwd_off, np.int32, nid + 1).copy(),
                             _view(out.fwd_cand, np.int32, nf).copy(),
                             _view(out.rev_off, np.int32, nid + 1).copy(),
                             _view(out.rev_cand, np.int32, nr).copy())

    def seen_tokens(self) -> tuple[list[str], list[str]]:
        """Normalized token strings of the last emit's source / target sentences."""
        out = []
        for which in (0, 1):
            p, n = C.c_void_p(), C.c_int64()
            N.check(self._lib.bm_ingest_seen(self._h, which, C.byref(p), C.byref(n)))
            raw = _bytes_at(p, n.value)
            out.append(raw.decode("utf-8").split("\0")[:-1] if raw else [])
        return out[0], out[1]

    def norm_keys(self) -> np.ndarray:
        """Per sentence, an id of its normalized text (bm_merge_bidir's key)."""
        p = C.c_void_p()
        N.check(self._lib.bm_ingest_norm_keys(self._h, C.byref(p)))
        return _view(p.value, np.int32, self.packed.n_sent)

    def emit_merged(self, recs: np.ndarray, skip: np.ndarray) -> tuple[bytes, list[int]]:
        """TSV bytes + report of device-merged records (bm_ingest_emit_merged)."""
        recs = np.ascontiguousarray(recs)
        sk = np.ascontiguousarray(skip, dtype=np.uint8)
        out = C.c_char_p()
        olen = C.c_int64()
        rep = np.zeros(6, dtype=np.int64)
        N.check(self._lib.bm_ingest_emit_merged(self._h, recs.ctypes.data, recs.shape[0],
                                                sk.ctypes.data, C.byref(out), C.byref(olen),
                                                rep.ctypes.data))
        data = _bytes_at(out, olen.value)
        return data, rep.tolist()

    def emit(self, fwd: np.ndarray, bwd: np.ndarray | None, swap_f: np.ndarray,
             swap_b: np.ndarray, skip: np.ndarray) -> tuple[bytes, list[int]]:
        fwd = np.ascontiguousarray(fwd)
        b = np.ascontiguousarray(bwd) if bwd is not None else fwd[:0]
        sf = np.ascontiguousarray(swap_f, dtype=np.uint8)
        sb = np.ascontiguousarray(swap_b, dtype=np.uint8)
        sk = np.ascontiguousarray(skip, dtype=np.uint8)
        out = C.c_char_p()
        olen = C.c_int64()
        rep = np.zeros(6, dtype=np.int64)
        N.check(self._lib.bm_ingest_emit(self._h, fwd.ctypes.data, fwd.shape[0], b.ctypes.data,
                                         b.shape[0], int(bwd is not None), sf.ctypes.data,
                                         sb.ctypes.data, sk.ctypes.data, C.byref(out),
                                         C.byref(olen), rep.ctypes.data))
        data = _bytes_at(out, olen.value)
        return data, rep.tolist()


def _orientations(langs, model: ClassifierModel, lex: Lexicon) -> np.ndarray | None:
    """Per-doc swapped flags (miner.py _orientation), or None when any
    document would raise DataError (the Python path then reproduces it)."""
    direction = tuple(model.direction)
    if tuple(lex.direction) != direction:
        return None
    out = np.zeros(len(langs), dtype=np.uint8)
    for k, (sl, tl) in enumerate(langs):
        if (sl, tl) == direction:
            continue
        if (tl, sl) == direction:
            out[k] = 1
            continue
        return None
    return out


# streamed files: chunks of about this many bytes are ingested, mined and
# emitted in turn (the next chunk is ingested on a host thread meanwhile)
CHUNK_BYTES = 256 << 20


def _chunk_cuts(path: str, chunk: int) -> list[int]:
    """Byte offsets of line starts splitting the file into ~chunk-byte pieces
    (cuts after a newline byte; a file without one stays whole)."""
    import os

    size = os.path.getsize(path)
    cuts = [0]
    with open(path, "rb") as fh:
        pos = chunk
        while pos < size:
            fh.seek(pos)
            buf = fh.read(1 << 16)
            k = buf.find(b"\n")
            while k < 0 and buf:
                pos += len(buf)
                buf = fh.read(1 << 16)
                k = buf.find(b"\n")
            if k < 0:
                break
            cut = pos + k + 1
            if cut >= size:
                break
            cuts.append(cut)
            pos = cut + chunk
    cuts.append(size)
    return cuts


def mine_corpus_file(
    docs_path: str,
    forward: ClassifierModel,
    backward: ClassifierModel | None,
    lex: Lexicon,
    cfg,
    out: IO[str],
    on_skip: Callable[[str, str], None] | None = None,
):
    """``mine_corpus(load_document_pairs(docs_path, on_skip=on_skip), ...)``
    with the native reader, lexicon lowering, merge and TSV emission, streamed
    in chunks of CHUNK_BYTES: each chunk's TSV is written before the next is
    mined. A chunk the native path cannot reproduce exactly (see the module
    docstring) hands the rest of the file, from its first line, to the Python
    reader -- the output up to there is the same either way."""
    import os
    from concurrent.futures import ThreadPoolExecutor

    from . import aligner, engine
    from .corpus import _iter_pairs
    from .miner import MiningReport, _mine_stream

    start = time.perf_counter()
    LAST_TIMINGS.clear()
    for k in ("ingest", "lexicon", "mine", "emit", "write"):
        LAST_TIMINGS[k] = 0.0
    report = MiningReport()
    src_tok: set[str] = set()
    tgt_tok: set[str] = set()
    if backward is not None:
        lex.reversed()
    chunk = int(os.environ.get("BM_STREAM_CHUNK_BYTES", CHUNK_BYTES))
    cuts = _chunk_cuts(docs_path, max(chunk, 1))
    LAST_TIMINGS["chunks"] = len(cuts) - 1

    def load(q: int, line0: int):
        t = time.perf_counter()
        nc = NativeCorpus.load_range(docs_path, cuts[q], cuts[q + 1], line0)
        return nc, time.perf_counter() - t

    def python_rest(line0: int):
        _mine_stream(_iter_pairs(docs_path, on_skip, line0), forward, backward, lex, cfg, out,
                     report, src_tok, tgt_tok)

    def finish():
        report.unique_src_tokens = len(src_tok)
        report.unique_tgt_tokens = len(tgt_tok)
        report.wall_clock_seconds = time.perf_counter() - start
        return report

    line0 = 0
    with ThreadPoolExecutor(max_workers=1) as pool:
        nxt = pool.submit(load, 0, 0)
        for q in range(len(cuts) - 1):
            nc, dt = nxt.result()
            LAST_TIMINGS["ingest"] += dt
            ok = nc is not None
            if ok:
                sw_f = _orientations(nc.langs, forward, lex)
                sw_b = None
                if backward is not None and sw_f is not None:
                    sw_b = _orientations(nc.langs, backward, lex.reversed())
                    ok = sw_b is not None
                ok = ok and sw_f is not None
            if not ok:
                python_rest(line0)
                return finish()
            if q + 2 < len(cuts):  # the next chunk is read while this one is mined
                nxt = pool.submit(load, q + 1, line0 + nc.n_lines)
            _mine_chunk(nc, forward, backward, lex, cfg, out, on_skip, sw_f, sw_b, report,
                        src_tok, tgt_tok, aligner, engine)
            line0 += nc.n_lines
    return finish()


def _mine_chunk(nc, forward, backward, lex, cfg, out, on_skip, sw_f, sw_b, report, src_tok,
                tgt_tok, aligner, engine) -> None:
    if sw_b is None:
        sw_b = np.zeros_like(sw_f)
    for _ln, pid, side in nc.skipped:
        log.warning("skipping pair %r: empty %s document", pid, side)
        if on_skip is not None:
            on_skip(pid, f"empty {side} document")
    c = nc.packed
    n = c.n.astype(np.int64)
    m = c.m.astype(np.int64)
    over = n * m > aligner.MAX_CELLS
    skip = over.astype(np.uint8)
    for k in np.nonzero(skip)[0].tolist():
        a, b = (int(c.m[k]), int(c.n[k])) if sw_f[k] else (int(c.n[k]), int(c.m[k]))
        why = (f"document pair {nc.doc_ids[k]!r} needs a {a}x{b} matrix, "
               f"over the {aligner.MAX_CELLS} cell limit")
        log.warning("skipping: %s", why)
    work = np.nonzero(skip == 0)[0].astype(np.int64)
    rec_dtype = np.dtype(N.RECORD_DTYPE)
    fwd = np.zeros(0, dtype=rec_dtype)
    bwd = None if backward is None else np.zeros(0, dtype=rec_dtype)
    merged = None
    t0 = time.perf_counter()
    if work.size:
        plex = nc.lexicon(lex)
        LAST_TIMINGS["lexicon"] += time.perf_counter() - t0
        dc = engine.DeviceCorpus.upload(c)
        idx = work.tolist()

        def run(model, pl, swapped):
            dl = engine.DeviceLexicon.upload(pl)
            view = engine.DocView.of(c, idx, [bool(x) for x in swapped[work]])
            return engine.mine_device(dc, dl, view, model, cfg.params.threshold,
                                      cfg.params.penalty)

        f, nf, _ = run(forward, plex, sw_f)
        if backward is None:
            fwd = engine.to_host(f[: nf * 24]).view(rec_dtype).copy()
            fwd["doc"] = work[fwd["doc"]]
        else:
            # bidirectional_merge on the device (bm_merge_bidir), keyed on the
            # native reader's normalized-text ids
            b, nb, _ = run(backward, plex.swapped(), sw_b)
            merged = engine.merge_bidir(f, nf, b, nb, c.src0[work], c.tgt0[work],
                                        engine.to_dev(nc.norm_keys(), engine.device()),
                                        sw_f[work], sw_b[work]).copy()
            merged["doc"] = work[merged["doc"]]
    t1 = time.perf_counter()
    LAST_TIMINGS["mine"] += t1 - t0
    if merged is not None:
        data, rep = nc.emit_merged(merged, skip)
    else:
        data, rep = nc.emit(fwd, bwd, sw_f, sw_b, skip)
    src, tgt = nc.seen_tokens()
    src_tok.update(src)
    tgt_tok.update(tgt)
    t2 = time.perf_counter()
    out.write(data.decode("utf-8"))
    LAST_TIMINGS["emit"] += t2 - t1
    LAST_TIMINGS["write"] += time.perf_counter() - t2
    report.pairs_emitted += rep[0]
    report.per_direction["forward"] += rep[1]
    report.per_direction["backward"] += rep[2]
    report.docs_processed += rep[5]
    report.docs_skipped += int(skip.sum())
