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
