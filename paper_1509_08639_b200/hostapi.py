"""End-to-end call through the C ABI with HOST buffers (bm_mine_host).

This is what a foreign binding of the reference's mining API would call: the
packed corpus, lexicon and model live in host memory; one call copies them to
the GPU, mines every document, compacts the records and copies them back in
document order. ``PinnedBatch`` stages the arrays in page-locked memory once
so the per-call H2D copies run at full PCIe/C2C bandwidth.
"""

from __future__ import annotations

import ctypes as C

import numpy as np

from . import _native as N
from .pack import PackedCorpus, PackedLexicon

_SENT = ("n_tok", "n_punct", "n_alpha", "tok_off", "tok_id", "tok_alpha", "dig_off", "dig_id")
_DOCS = ("src0", "n", "tgt0", "m")
_LEX = ("fwd_off", "fwd_cand", "rev_off", "rev_cand")


def _pinned(a: np.ndarray) -> tuple[object, np.ndarray]:
    import torch

    a = np.ascontiguousarray(a)
    t = torch.empty(a.nbytes, dtype=torch.uint8, pin_memory=True)
    view = t.numpy().view(a.dtype).reshape(a.shape)
    view[...] = a
    return t, view


def wire_ok(corpus: PackedCorpus, plex: PackedLexicon) -> bool:
    """The compact wire format holds this batch (16-bit ids, 8-bit counts)."""
    return (plex.n_ids <= 65536 and corpus.n_sent > 0
            and int(corpus.n_tok.max(initial=0)) <= 255
            and int(corpus.tok_alpha.max(initial=0)) <= 255)


def packed_ok(corpus: PackedCorpus, plex: PackedLexicon) -> bool:
    """The packed format holds this batch (14-bit ids, alphabetic counts <= 3)."""
    return (plex.n_ids <= 16384 and corpus.n_sent > 0
            and int(corpus.n_tok.max(initial=0)) <= 255
            and int(corpus.tok_alpha.max(initial=0)) <= 3)


def to_wire(corpus: PackedCorpus) -> dict[str, np.ndarray]:
    return {
        "n_tok": corpus.n_tok.astype(np.uint8), "n_punct": corpus.n_punct.astype(np.uint8),
        "n_alpha": corpus.n_alpha.astype(np.uint8), "tok_off": corpus.tok_off,
        "tok_id": corpus.tok_id.astype(np.uint16), "tok_alpha": corpus.tok_alpha.astype(np.uint8),
        "dig_off": corpus.dig_off, "dig_id": corpus.dig_id.astype(np.uint16),
    }


_PACKED = ("tok_off", "dig_off", "counts", "tok_off32", "dig_off32", "tok_pk", "dig_id")


def to_packed(corpus: PackedCorpus) -> dict[str, np.ndarray]:
    """bm_wire_packed arrays (include/bimine_b200.h)."""
    to, do = corpus.tok_off, corpus.dig_off
    counts = (corpus.n_tok.astype(np.uint32) | corpus.n_punct.astype(np.uint32) << 8
              | np.diff(to).astype(np.uint32) << 16 | np.diff(do).astype(np.uint32) << 24)
    return {
        "tok_off": to, "dig_off": do, "counts": counts,
        "tok_off32": np.ascontiguousarray(to[::32]), "dig_off32": np.ascontiguousarray(do[::32]),
        "tok_pk": (corpus.tok_id.astype(np.uint16) << 2) | corpus.tok_alpha.astype(np.uint16),
        "dig_id": corpus.dig_id.astype(np.uint16),
    }


class PinnedBatch:
    """Packed arrays copied once into page-locked host memory + C structs.

    wire=True stages the most compact host format the batch fits: the packed
    format (bm_mine_host_packed, ~0.6x the wire bytes) or the wire format
    (bm_mine_host_wire, ~half the plain bytes); wire="wire" / "packed" picks
    one; wire=False sends the plain bm_sentences arrays (bm_mine_host).
    ``h2d_bytes`` counts the bytes one call copies host -> device.
    """

    def __init__(self, corpus: PackedCorpus, plex: PackedLexicon, pin: bool = True,
                 wire: bool | str = True):
        self.keep = []
        if wire is True:
            fmt = ("packed" if packed_ok(corpus, plex) else
                   "wire" if wire_ok(corpus, plex) else "full")
        elif wire in ("packed", "wire"):
            fmt = wire
            ok = packed_ok if wire == "packed" else wire_ok
            if not ok(corpus, plex):
                raise ValueError(f"the batch does not fit the {wire} format")
        else:
            fmt = "full"
        self.fmt = fmt
        self.wire = fmt != "full"
        if fmt == "packed":
            src, names = to_packed(corpus), _PACKED
        elif fmt == "wire":
            src, names = to_wire(corpus), _SENT
        else:
            src, names = {k: getattr(corpus, k) for k in _SENT}, _SENT
        arrs = {name: src[name] for name in names}
        for name in _DOCS:
            arrs[name] = getattr(corpus, name)
        for name in _LEX:
            arrs[name] = getattr(plex, name)
        self.h2d_bytes = 0
        for k, v in arrs.items():
            if pin:
                t, view = _pinned(v)
                self.keep.append(t)
            else:
                view = np.ascontiguousarray(v)
            arrs[k] = view
            self.keep.append(view)
            if not (fmt == "packed" and k in ("tok_off", "dig_off")):  # planning only
                self.h2d_bytes += view.nbytes
        self.arrs = arrs
        cls = {"packed": N.WirePacked, "wire": N.Wire, "full": N.Sentences}[fmt]
        self.sent = cls(corpus.n_sent, *[arrs[k].ctypes.data for k in names])
        self.docs = N.Docs(corpus.n_docs, *[arrs[k].ctypes.data for k in _DOCS])
        self.lex = N.LexiconC(plex.n_ids, *[arrs[k].ctypes.data for k in _LEX])
        n, m = arrs["n"], arrs["m"]
        self.rec_cap = int(np.minimum(n, m).clip(min=0).sum())
        self.n_docs = corpus.n_docs
        if pin:
            self.rec_t, self.rec = _pinned(np.zeros(max(self.rec_cap, 1), dtype=np.dtype(N.RECORD_DTYPE)))
            self.cost_t, self.cost = _pinned(np.zeros(max(self.n_docs, 1), dtype=np.float64))
        else:
            self.rec = np.zeros(max(self.rec_cap, 1), dtype=np.dtype(N.RECORD_DTYPE))
            self.cost = np.zeros(max(self.n_docs, 1), dtype=np.float64)


def mine_pinned(pb: PinnedBatch, model, threshold: float, penalty: float, stream: int = 0):
    """One bm_mine_host call; returns (records view, n_records, d2h bytes)."""
    lib = N.lib()
    n_rec = C.c_int64(0)
    fn = {"packed": lib.bm_mine_host_packed, "wire": lib.bm_mine_host_wire,
          "full": lib.bm_mine_host}[pb.fmt]
    N.check(fn(C.byref(pb.sent), C.byref(pb.docs), C.byref(pb.lex),
               C.byref(N.model_struct(model)), float(threshold), float(penalty),
               pb.rec.ctypes.data, pb.rec_cap, C.byref(n_rec), pb.cost.ctypes.data, stream))
    k = n_rec.value
    d2h = k * 24 + pb.n_docs * 8 + 8
    return pb.rec[:k], k, d2h


def mine_host(corpus: PackedCorpus, plex: PackedLexicon, model, threshold: float, penalty: float,
              wire: bool | str = False, pin: bool = False):
    """One call with host buffers; pin=True stages them page-locked (records are
    then written by the GPU straight into the pinned output buffer)."""
    pb = PinnedBatch(corpus, plex, pin=pin, wire=wire)
    recs, k, _ = mine_pinned(pb, model, threshold, penalty)
    return recs.copy(), pb.cost[: pb.n_docs].copy()


class TunePinned:
    """A tuning dev set staged page-locked once (tuner.py:112-154 inputs): the
    packed sentences, the documents' ranges and the packed gold keys
    (engine.pack_gold). ``tune_pinned`` copies it to the GPU chunk by chunk,
    each chunk's copy overlapping the sweep of the chunk before."""

    def __init__(self, corpus: PackedCorpus, gold_keys: np.ndarray, gold_off: np.ndarray):
        self.corpus = corpus
        self.n_docs = int(corpus.n_docs)
        self.host = {k: _pinned(getattr(corpus, k)) for k in _SENT}
        self.docs = {k: _pinned(np.asarray(getattr(corpus, k), dtype=np.int32)) for k in _DOCS}
        self.gold = (_pinned(np.asarray(gold_keys, dtype=np.int64)),
                     _pinned(np.asarray(gold_off, dtype=np.int64)))
        self.max_tok = int(corpus.n_tok.max(initial=0))
        self.h2d_bytes = (sum(v[1].nbytes for v in self.host.values())
                          + sum(v[1].nbytes for v in self.docs.values())
                          + self.gold[0][1].nbytes + self.gold[1][1].nbytes)
        self._dev = None
        n = self.docs["n"][1].astype(np.int64)
        m = self.docs["m"][1].astype(np.int64)
        s_end = np.maximum(self.docs["src0"][1] + n, self.docs["tgt0"][1] + m)
        # sentences [0, hi_k) must be resident before documents < d1 of chunk k run
        self._hi = np.maximum.accumulate(s_end) if self.n_docs else s_end
        self._cells = np.cumsum(n * m)

    def chunks(self, n_chunks: int):
        """[d0, d1) ranges: a small first chunk (the GPU starts early), then
        equal cell counts."""
        if self.n_docs == 0:
            return []
        total = int(self._cells[-1])
        first = total / (4 * n_chunks)
        cuts = [first + (total - first) * k / n_chunks for k in range(n_chunks)]
        ends = sorted({int(np.searchsorted(self._cells, c, side="left")) + 1 for c in cuts})
        ends = [min(e, self.n_docs) for e in ends] + [self.n_docs]
        out, d0 = [], 0
        for e in ends:
            if e > d0:
                out.append((d0, e))
                d0 = e
        return out

    def device_buffers(self):
        if self._dev is None:
            import torch

            dev = torch.device("cuda", torch.cuda.current_device())
            mk = lambda v: torch.empty(max(v[1].nbytes, 1), dtype=torch.uint8, device=dev)  # noqa: E731
            self._dev = ({k: mk(v) for k, v in self.host.items()},
                         {k: mk(v) for k, v in self.docs.items()},
                         (mk(self.gold[0]), mk(self.gold[1])))
        return self._dev


_STREAMS = {}


def _private_streams():
    """(work, copy) streams of the current device for tune_pinned. The sweep
    runs on its own stream, not the caller's: the caller's is usually the
    legacy default stream, which would order every copy-stream operation
    against the sweep and serialise the copies with the kernels."""
    import torch

    d = torch.cuda.current_device()
    if d not in _STREAMS:
        _STREAMS[d] = (torch.cuda.Stream(device=d), torch.cuda.Stream(device=d))
    return _STREAMS[d]


def tune_pinned(tp: TunePinned, dl, model, penalties, thresholds, n_chunks: int | None = None):
    """tune's counting sweep end to end from page-locked host buffers: chunk k's
    sentences, documents and gold keys are copied on a copy stream one chunk
    ahead of the bm_tune call of chunk k - 1 on the current stream (so the
    sweep's own small plan uploads never queue behind the whole dev set's
    bulk copy), and every chunk's pred/hit counts add into the same device
    totals (bm_tune accumulates). Returns (pred, hit) [n_pen, n_thr] int64 on
    the host."""
    import torch

    from . import engine

    import os

    if n_chunks is None:
        n_chunks = int(os.environ.get("BM_TUNE_CHUNKS", "6"))
    lib = N.lib()
    sent_d, docs_d, (gk_d, go_d) = tp.device_buffers()
    caller = torch.cuda.current_stream()
    main, cs = _private_streams()
    main.wait_stream(caller)
    pen = np.ascontiguousarray(np.asarray(penalties, dtype=np.float64))
    thr = np.asarray(thresholds, dtype=np.float64)
    dev = sent_d["n_tok"].device
    with torch.cuda.stream(main):
        pred = torch.zeros((len(pen), len(thr)), dtype=torch.int64, device=dev)
        hit = torch.zeros((len(pen), len(thr)), dtype=torch.int64, device=dev)
        thr_d = torch.from_numpy(thr).pin_memory().to(dev, non_blocking=True)
    c = tp.corpus
    tok_off, dig_off = tp.host["tok_off"][1], tp.host["dig_off"][1]
    goff = tp.gold[1][1]
    cs.wait_stream(main)  # the device buffers are free once earlier work on main is done

    def cp(dst, src, lo, hi):
        if hi > lo:
            isz = src[1].itemsize
            dst[lo * isz: hi * isz].copy_(src[0][lo * isz: hi * isz], non_blocking=True)

    state = {"hi": 0}
    events = []

    def enqueue_copy(d0, d1):
        with torch.cuda.stream(cs):
            if not events:  # the documents' ranges, once
                for k in _DOCS:
                    cp(docs_d[k], tp.docs[k], 0, tp.n_docs)
            a, b = state["hi"], int(tp._hi[d1 - 1])
            if b > a:
                for k in ("n_tok", "n_punct", "n_alpha"):
                    cp(sent_d[k], tp.host[k], a, b)
                cp(sent_d["tok_off"], tp.host["tok_off"], a, b + 1)
                cp(sent_d["dig_off"], tp.host["dig_off"], a, b + 1)
                e0, e1 = int(tok_off[a]), int(tok_off[b])
                cp(sent_d["tok_id"], tp.host["tok_id"], e0, e1)
                cp(sent_d["tok_alpha"], tp.host["tok_alpha"], e0, e1)
                cp(sent_d["dig_id"], tp.host["dig_id"], int(dig_off[a]), int(dig_off[b]))
                state["hi"] = b
            cp(go_d, tp.gold[1], d0, d1 + 1)
            cp(gk_d, tp.gold[0], int(goff[d0]), int(goff[d1]))
            ev = torch.cuda.Event()
            ev.record(cs)
            events.append(ev)

    sent = N.Sentences(c.n_sent, *[int(sent_d[k].data_ptr()) for k in _SENT])
    chunks = tp.chunks(n_chunks)
    if chunks:
        enqueue_copy(*chunks[0])
    n_h = tp.docs["n"][1]
    m_h = tp.docs["m"][1]
    for q, (d0, d1) in enumerate(chunks):
        if q + 1 < len(chunks):
            enqueue_copy(*chunks[q + 1])
        main.wait_event(events[q])
        docs = N.Docs(d1 - d0, *[int(docs_d[k].data_ptr()) + 4 * d0 for k in _DOCS])
        nh = np.ascontiguousarray(n_h[d0:d1])
        mh = np.ascontiguousarray(m_h[d0:d1])
        N.check(lib.bm_tune(C.byref(sent), C.byref(docs), nh.ctypes.data, mh.ctypes.data,
                            C.byref(dl.lex), C.byref(N.model_struct(model)), pen.ctypes.data,
                            len(pen), engine._ptr(thr_d), len(thr), int(gk_d.data_ptr()),
                            int(go_d.data_ptr()) + 8 * d0, engine._ptr(pred), engine._ptr(hit),
                            tp.max_tok, int(main.cuda_stream)))
    main.wait_stream(cs)
    caller.wait_stream(main)
    with torch.cuda.stream(main):
        out = pred.cpu().numpy(), hit.cpu().numpy()
    return out
