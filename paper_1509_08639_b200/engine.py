"""Batched device execution of the hot path through the C ABI.

torch provides device memory, the current stream and (for multi-GPU) the
process group; every byte of hot-path arithmetic runs in libbimine_b200.so.
"""

from __future__ import annotations

import ctypes as C
from dataclasses import dataclass

import numpy as np

from . import _native as N
from .pack import PackedCorpus, PackedLexicon

_torch = None


def torch_mod():
    global _torch
    if _torch is None:
        import torch

        _torch = torch
    return _torch


def device():
    torch = torch_mod()
    N.lib()  # raises NativeUnavailableError without a GPU / library
    if not torch.cuda.is_available():
        raise N.NativeUnavailableError("torch sees no CUDA device")
    return torch.device("cuda", torch.cuda.current_device())


def stream_ptr() -> int:
    return int(torch_mod().cuda.current_stream().cuda_stream)


def _ptr(t) -> int:
    return int(t.data_ptr()) if t is not None and t.numel() > 0 else 0


def to_host(t) -> np.ndarray:
    """Device tensor -> numpy. Large results land in page-locked memory from
    torch's caching host allocator and are returned as a view of it: a plain
    .cpu() copies into freshly faulted pageable pages (C3's 127 MB of records
    took 60 ms that way, 2 GB/s)."""
    torch = torch_mod()
    if not t.is_cuda or t.numel() * t.element_size() < (1 << 20):
        return t.cpu().numpy()
    host = torch.empty(t.shape, dtype=t.dtype, pin_memory=True)
    host.copy_(t)
    return host.numpy()  # keeps `host` alive


def to_dev(a: np.ndarray, dev):
    torch = torch_mod()
    a = np.ascontiguousarray(a)
    if not a.flags.writeable:  # views of native buffers: torch wants writable memory
        a = a.copy()
    if a.dtype == np.uint16:  # move unsigned arrays as raw bytes of the signed type
        t = torch.from_numpy(a.view(np.int16))
    elif a.dtype == np.uint32:
        t = torch.from_numpy(a.view(np.int32))
    else:
        t = torch.from_numpy(a)
    return t.to(dev, non_blocking=False)


@dataclass
class DeviceCorpus:
    """Packed sentences resident in HBM plus the bm_sentences view."""

    corpus: PackedCorpus
    tensors: dict
    sent: N.Sentences
    max_tok: int = 0  # largest token count T of any sentence (routing input)

    @classmethod
    def upload(cls, corpus: PackedCorpus) -> "DeviceCorpus":
        dev = device()
        names = ("n_tok", "n_punct", "n_alpha", "tok_off", "tok_id", "tok_alpha", "dig_off",
                 "dig_id")
        t = {k: to_dev(getattr(corpus, k), dev) for k in names}
        sent = N.Sentences(corpus.n_sent, *[_ptr(t[k]) for k in names])
        return cls(corpus, t, sent, int(corpus.n_tok.max(initial=0)))

    def doc_token_max(self, view: "DocView") -> np.ndarray:
        """Per-doc max T of the view's docs (bm_mine's routing input). When no
        sentence of the corpus exceeds 255 tokens the bound is all a doc needs,
        so the per-doc scan is skipped; otherwise it is computed once per view."""
        if self.max_tok <= 255:
            return np.full(len(view.n), self.max_tok, dtype=np.int32)
        return view.token_max(self.corpus)


@dataclass
class DeviceLexicon:
    plex: PackedLexicon
    tensors: dict
    lex: N.LexiconC

    @classmethod
    def upload(cls, plex: PackedLexicon) -> "DeviceLexicon":
        dev = device()
        names = ("fwd_off", "fwd_cand", "rev_off", "rev_cand")
        t = {k: to_dev(getattr(plex, k), dev) for k in names}
        return cls(plex, t, N.LexiconC(plex.n_ids, *[_ptr(t[k]) for k in names]))


@dataclass
class DocView:
    """A list of (source range, target range) pairs over a DeviceCorpus."""

    src0: np.ndarray
    n: np.ndarray
    tgt0: np.ndarray
    m: np.ndarray
    tensors: dict
    docs: N.Docs

    @classmethod
    def upload(cls, src0, n, tgt0, m) -> "DocView":
        dev = device()
        arrs = {"src0": _i32(src0), "n": _i32(n), "tgt0": _i32(tgt0), "m": _i32(m)}
        t = {k: to_dev(v, dev) for k, v in arrs.items()}
        docs = N.Docs(len(arrs["n"]), _ptr(t["src0"]), _ptr(t["n"]), _ptr(t["tgt0"]), _ptr(t["m"]))
        return cls(arrs["src0"], arrs["n"], arrs["tgt0"], arrs["m"], t, docs)

    @classmethod
    def of(cls, corpus: PackedCorpus, idx=None, swapped=None) -> "DocView":
        """Docs ``idx`` of the corpus; swapped[k] exchanges source and target."""
        idx = np.arange(corpus.n_docs) if idx is None else np.asarray(idx, dtype=np.int64)
        s0, n, t0, m = corpus.src0[idx], corpus.n[idx], corpus.tgt0[idx], corpus.m[idx]
        if swapped is not None:
            sw = np.asarray(swapped, dtype=bool)
            s0, t0 = np.where(sw, t0, s0), np.where(sw, s0, t0)
            n, m = np.where(sw, m, n), np.where(sw, n, m)
        return cls.upload(s0, n, t0, m)

    def token_max(self, corpus: PackedCorpus) -> np.ndarray:
        cached = getattr(self, "_tmax", None)
        if cached is not None and cached[0] is corpus:
            return cached[1]
        view = PackedCorpus(corpus.n_tok, corpus.n_punct, corpus.n_alpha, corpus.tok_off,
                            corpus.tok_id, corpus.tok_alpha, corpus.dig_off, corpus.dig_id,
                            self.src0, self.n, self.tgt0, self.m)
        out = view.doc_token_max()
        self._tmax = (corpus, out)
        return out


def _i64(x) -> np.ndarray:
    return np.ascontiguousarray(np.asarray(x, dtype=np.int64))


def _i32(x) -> np.ndarray:
    return np.ascontiguousarray(np.asarray(x, dtype=np.int32))


def score(dc: DeviceCorpus, dl: DeviceLexicon, view: DocView, model):
    """K1 for every doc of the view -> (S device buffer, offsets, pitch, ...)."""
    torch = torch_mod()
    lib = N.lib()
    docs, lex, n, m = view.docs, dl.lex, view.n, view.m
    pitch = _i32((m + 3) // 4 * 4)
    sizes = n.astype(np.int64) * pitch
    s_off = np.zeros(len(n), dtype=np.int64)
    if len(n) > 1:
        s_off[1:] = np.cumsum(sizes)[:-1]
    total = int(sizes.sum())
    dev = device()
    S = torch.empty(max(total, 1), dtype=torch.float64, device=dev)
    s_off_d, pitch_d = to_dev(s_off, dev), to_dev(pitch, dev)
    n_h, m_h = _i32(n), _i32(m)
    N.check(lib.bm_score(C.byref(dc.sent), C.byref(docs), n_h.ctypes.data, m_h.ctypes.data,
                         C.byref(lex), C.byref(N.model_struct(model)), _ptr(s_off_d),
                         _ptr(pitch_d), _ptr(S), stream_ptr()))
    return S, s_off, pitch, s_off_d, pitch_d


def matrices_from_buffer(S, s_off, pitch, n, m) -> list[np.ndarray]:
    host = to_host(S)
    out = []
    for k in range(len(n)):
        o, p, nn, mm = int(s_off[k]), int(pitch[k]), int(n[k]), int(m[k])
        out.append(np.ascontiguousarray(host[o : o + nn * p].reshape(nn, p)[:, :mm]))
    return out


def upload_matrices(mats: list[np.ndarray]):
    """Copy host similarity matrices into one pitched device buffer."""
    torch = torch_mod()
    dev = device()
    n = _i32([a.shape[0] for a in mats])
    m = _i32([a.shape[1] for a in mats])
    pitch = _i32((m + 3) // 4 * 4)
    sizes = n.astype(np.int64) * pitch
    s_off = np.zeros(len(mats), dtype=np.int64)
    if len(mats) > 1:
        s_off[1:] = np.cumsum(sizes)[:-1]
    host = np.zeros(max(int(sizes.sum()), 1), dtype=np.float64)
    for k, a in enumerate(mats):
        o, p = int(s_off[k]), int(pitch[k])
        host[o : o + a.shape[0] * p].reshape(a.shape[0], p)[:, : a.shape[1]] = a
    S = torch.from_numpy(host).to(dev)
    return S, s_off, pitch, n, m


def nw_paths(S, s_off, pitch, n, m, penalty: float):
    """K2/K3 + K4a: costs and move lists (forward order) for each matrix."""
    torch = torch_mod()
    lib = N.lib()
    dev = device()
    k = len(n)
    words = np.array([lib.bm_dirs_words(int(a), int(b)) for a, b in zip(n, m)], dtype=np.int64)
    dir_off = np.zeros(k, dtype=np.int64)
    if k > 1:
        dir_off[1:] = np.cumsum(words)[:-1]
    dirs = torch.empty(max(int(words.sum()), 1), dtype=torch.int32, device=dev)
    cost = torch.empty(k, dtype=torch.float64, device=dev)
    n_h, m_h = _i32(n), _i32(m)
    n_d, m_d = to_dev(n_h, dev), to_dev(m_h, dev)
    s_off_d, pitch_d, dir_off_d = to_dev(_i64(s_off), dev), to_dev(_i32(pitch), dev), to_dev(dir_off, dev)
    N.check(lib.bm_nw(_ptr(S), _ptr(s_off_d), _ptr(pitch_d), _ptr(n_d), _ptr(m_d),
                      n_h.ctypes.data, m_h.ctypes.data, k, float(penalty), _ptr(dirs),
                      _ptr(dir_off_d), _ptr(cost), stream_ptr()))
    cap = (n_h.astype(np.int64) + m_h)
    mv_off = np.zeros(k, dtype=np.int64)
    if k > 1:
        mv_off[1:] = np.cumsum(cap)[:-1]
    tot = max(int(cap.sum()), 1)
    op = torch.empty(tot, dtype=torch.int8, device=dev)
    mi = torch.empty(tot, dtype=torch.int32, device=dev)
    mj = torch.empty(tot, dtype=torch.int32, device=dev)
    ln = torch.empty(k, dtype=torch.int32, device=dev)
    mv_off_d = to_dev(mv_off, dev)
    N.check(lib.bm_traceback(_ptr(dirs), _ptr(dir_off_d), _ptr(n_d), _ptr(m_d), k, _ptr(mv_off_d),
                             _ptr(op), _ptr(mi), _ptr(mj), _ptr(ln), stream_ptr()))
    op_h, mi_h, mj_h, ln_h = op.cpu().numpy(), mi.cpu().numpy(), mj.cpu().numpy(), ln.cpu().numpy()
    paths = []
    for q in range(k):
        o, L = int(mv_off[q]), int(ln_h[q])
        paths.append((op_h[o : o + L][::-1], mi_h[o : o + L][::-1], mj_h[o : o + L][::-1]))
    return cost.cpu().numpy(), paths


def record_offsets(n: np.ndarray, m: np.ndarray) -> np.ndarray:
    cap = np.minimum(n, m).astype(np.int64).clip(min=0)
    off = np.zeros(len(n), dtype=np.int64)
    if len(n) > 1:
        off[1:] = np.cumsum(cap)[:-1]
    return off


def mine_device(dc: DeviceCorpus, dl: DeviceLexicon, view: DocView, model, threshold: float,
                penalty: float):
    """Mining of every doc of the view, records left on the device:
    (dense records uint8 tensor, record count, cost tensor)."""
    torch = torch_mod()
    lib = N.lib()
    dev = device()
    docs, lex, n, m = view.docs, dl.lex, view.n, view.m
    k = len(n)
    rec_off = record_offsets(n, m)
    cap = int(np.minimum(n, m).clip(min=0).sum())
    rec = torch.empty(max(cap, 1) * 24, dtype=torch.uint8, device=dev)
    cnt = torch.zeros(max(k, 1), dtype=torch.int32, device=dev)
    cost = torch.empty(max(k, 1), dtype=torch.float64, device=dev)
    rec_off_d = to_dev(rec_off, dev)
    amax = dc.doc_token_max(view)
    n_h, m_h, a_h = _i32(n), _i32(m), _i32(amax)
    N.check(lib.bm_mine(C.byref(dc.sent), C.byref(docs), n_h.ctypes.data, m_h.ctypes.data,
                        a_h.ctypes.data, C.byref(lex), C.byref(N.model_struct(model)),
                        float(threshold), float(penalty), _ptr(rec_off_d), _ptr(rec), _ptr(cnt),
                        _ptr(cost), stream_ptr()))
    dense = torch.empty(max(cap, 1) * 24, dtype=torch.uint8, device=dev)
    total = torch.zeros(1, dtype=torch.int64, device=dev)
    N.check(lib.bm_compact(_ptr(rec), _ptr(rec_off_d), _ptr(cnt), k, _ptr(dense), _ptr(total),
                           stream_ptr()))
    return dense, int(total.item()), cost[:k]


def merge_bidir(fwd, n_fwd: int, bwd, n_bwd: int, src0, tgt0, norm_key, swap_f, swap_b):
    """bidirectional_merge on the device (bm_merge_bidir) of two passes' dense
    records over the same documents: host records in (document, source index,
    target index) order in the pairs' own orientation, pad = 0 forward /
    1 backward."""
    torch = torch_mod()
    lib = N.lib()
    dev = device()
    k = len(src0)
    s0, t0 = to_dev(_i32(src0), dev), to_dev(_i32(tgt0), dev)
    sf = to_dev(np.ascontiguousarray(swap_f, dtype=np.uint8), dev)
    sb = to_dev(np.ascontiguousarray(swap_b, dtype=np.uint8), dev)
    out = torch.empty(max(n_fwd + n_bwd, 1) * 24, dtype=torch.uint8, device=dev)
    total = torch.zeros(1, dtype=torch.int64, device=dev)
    N.check(lib.bm_merge_bidir(_ptr(fwd), n_fwd, _ptr(bwd), n_bwd, k, _ptr(s0), _ptr(t0),
                               _ptr(norm_key), _ptr(sf), _ptr(sb), _ptr(out), _ptr(total),
                               stream_ptr()))
    tot = int(total.item())
    return to_host(out[: tot * 24]).view(np.dtype(N.RECORD_DTYPE))


def mine(dc: DeviceCorpus, dl: DeviceLexicon, view: DocView, model, threshold: float,
         penalty: float):
    """Fused mining of every doc of the view -> (records ndarray, cost ndarray).

    Records are in document order (``doc`` = index into the view), and in path
    order within a document.
    """
    torch = torch_mod()
    lib = N.lib()
    dev = device()
    docs, lex, n, m = view.docs, dl.lex, view.n, view.m
    k = len(n)
    rec_off = record_offsets(n, m)
    cap = int(np.minimum(n, m).clip(min=0).sum())
    rec = torch.empty(max(cap, 1) * 24, dtype=torch.uint8, device=dev)
    cnt = torch.zeros(max(k, 1), dtype=torch.int32, device=dev)
    cost = torch.empty(max(k, 1), dtype=torch.float64, device=dev)
    rec_off_d = to_dev(rec_off, dev)
    amax = dc.doc_token_max(view)
    n_h, m_h, a_h = _i32(n), _i32(m), _i32(amax)
    N.check(lib.bm_mine(C.byref(dc.sent), C.byref(docs), n_h.ctypes.data, m_h.ctypes.data,
                        a_h.ctypes.data, C.byref(lex), C.byref(N.model_struct(model)),
                        float(threshold), float(penalty), _ptr(rec_off_d), _ptr(rec), _ptr(cnt),
                        _ptr(cost), stream_ptr()))
    dense = torch.empty(max(cap, 1) * 24, dtype=torch.uint8, device=dev)
    total = torch.zeros(1, dtype=torch.int64, device=dev)
    N.check(lib.bm_compact(_ptr(rec), _ptr(rec_off_d), _ptr(cnt), k, _ptr(dense), _ptr(total),
                           stream_ptr()))
    tot = int(total.item())
    recs = to_host(dense[: tot * 24]).view(np.dtype(N.RECORD_DTYPE))
    return recs, cost[:k].cpu().numpy()


def pack_gold(gold_keys: list[np.ndarray]):
    """Per-doc ascending gold keys (i * m + j) -> (keys int64, offsets int64 [k+1]),
    packed with one vectorised sort (tuner.py:157-203 gold set, as device keys)."""
    lens = np.fromiter((len(g) for g in gold_keys), dtype=np.int64, count=len(gold_keys))
    goff = np.zeros(len(gold_keys) + 1, dtype=np.int64)
    np.cumsum(lens, out=goff[1:])
    if not lens.sum():
        return np.zeros(0, np.int64), goff
    keys = np.concatenate([np.asarray(g, dtype=np.int64).ravel() for g in gold_keys])
    step = np.diff(keys)
    inner = goff[1:-1]
    step[inner[(inner > 0) & (inner < keys.size)] - 1] = 0  # doc boundaries may descend
    if (step < 0).any():  # sort within docs: one sort of (doc << 40 | key)
        if keys.min() < 0 or keys.max() >= (1 << 40):
            raise ValueError("gold keys must lie in [0, 2**40)")
        owner = np.repeat(np.arange(len(gold_keys), dtype=np.int64), lens)
        keys = np.sort((owner << 40) | keys) & ((1 << 40) - 1)
    return np.ascontiguousarray(keys), goff


class DeviceGold:
    """Packed gold keys resident on the device (uploaded once per sweep)."""

    def __init__(self, keys: np.ndarray, goff: np.ndarray):
        dev = device()
        self.keys = to_dev(keys, dev)
        self.goff = to_dev(goff, dev)

    @classmethod
    def of(cls, gold_keys: list[np.ndarray]) -> "DeviceGold":
        return cls(*pack_gold(gold_keys))


def tune_counts_device(dc: DeviceCorpus, dl: DeviceLexicon, view: DocView, model, penalties,
                       thresholds, gold: DeviceGold):
    """K5 on device-resident inputs: pred/hit counts [n_pen, n_thr] as device tensors."""
    torch = torch_mod()
    lib = N.lib()
    dev = device()
    pen = np.ascontiguousarray(np.asarray(penalties, dtype=np.float64))
    thr = np.asarray(thresholds, dtype=np.float64)
    pred = torch.zeros((len(pen), len(thr)), dtype=torch.int64, device=dev)
    hit = torch.zeros((len(pen), len(thr)), dtype=torch.int64, device=dev)
    thr_d = to_dev(thr, dev)
    n_h, m_h = _i32(view.n), _i32(view.m)
    N.check(lib.bm_tune(C.byref(dc.sent), C.byref(view.docs), n_h.ctypes.data, m_h.ctypes.data,
                        C.byref(dl.lex), C.byref(N.model_struct(model)), pen.ctypes.data, len(pen),
                        _ptr(thr_d), len(thr), _ptr(gold.keys), _ptr(gold.goff), _ptr(pred),
                        _ptr(hit), dc.max_tok, stream_ptr()))
    return pred, hit


def tune_counts(dc: DeviceCorpus, dl: DeviceLexicon, view: DocView, model, penalties,
                thresholds, gold_keys: list[np.ndarray]):
    """K5: pred/hit counts [n_pen, n_thr] over the view's docs."""
    pred, hit = tune_counts_device(dc, dl, view, model, penalties, thresholds,
                                   DeviceGold.of(gold_keys))
    return pred.cpu().numpy(), hit.cpu().numpy()


def features(dc: DeviceCorpus, dl: DeviceLexicon, q_src, q_tgt, pos_s, pos_t) -> np.ndarray:
    torch = torch_mod()
    lib = N.lib()
    dev = device()
    k = len(q_src)
    out = torch.empty((max(k, 1), 7), dtype=torch.float64, device=dev)
    a, b = to_dev(_i32(q_src), dev), to_dev(_i32(q_tgt), dev)
    c = to_dev(np.asarray(pos_s, dtype=np.float64), dev)
    d = to_dev(np.asarray(pos_t, dtype=np.float64), dev)
    N.check(lib.bm_features(C.byref(dc.sent), C.byref(dl.lex), _ptr(a), _ptr(b), _ptr(c),
                            _ptr(d), k, _ptr(out), stream_ptr()))
    return out[:k].cpu().numpy()


def confidences(feats: np.ndarray, model) -> np.ndarray:
    torch = torch_mod()
    lib = N.lib()
    dev = device()
    f = to_dev(np.ascontiguousarray(feats, dtype=np.float64), dev)
    k = feats.shape[0]
    out = torch.empty(max(k, 1), dtype=torch.float64, device=dev)
    N.check(lib.bm_confidence(_ptr(f), k, C.byref(N.model_struct(model)), _ptr(out), stream_ptr()))
    return out[:k].cpu().numpy()
