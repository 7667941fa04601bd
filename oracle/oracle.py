"""CPU ORACLE -- TEST INFRASTRUCTURE ONLY (parity checker and CPU baseline).

ctypes wrapper of liboracle.so (bimine_oracle.c), a C restatement of the
reference hot path that calls the C library's exp (the one CPython's math.exp
uses). Only tests/, __graft_entry__.smoke() and bench.py's CPU-baseline legs
import this module; the product package never does.

The arrays it consumes are the packed layout of include/bimine_b200.h with
HOST pointers (paper_1509_08639_b200.pack produces them).
"""

from __future__ import annotations

import ctypes as C
import os
import subprocess

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
LIB = os.path.join(HERE, "liboracle.so")

_p = C.c_void_p


class _Sent(C.Structure):
    _fields_ = [("n_sent", C.c_int32), ("n_tok", _p), ("n_punct", _p), ("n_alpha", _p),
                ("tok_off", _p), ("tok_id", _p), ("tok_alpha", _p), ("dig_off", _p),
                ("dig_id", _p)]


class _Docs(C.Structure):
    _fields_ = [("n_docs", C.c_int32), ("src0", _p), ("n", _p), ("tgt0", _p), ("m", _p)]


class _Lex(C.Structure):
    _fields_ = [("n_ids", C.c_int32), ("fwd_off", _p), ("fwd_cand", _p), ("rev_off", _p),
                ("rev_cand", _p)]


RECORD = np.dtype([("doc", "<i4"), ("i", "<i4"), ("j", "<i4"), ("pad", "<i4"), ("conf", "<f8")])

_lib = None


def build() -> str:
    subprocess.check_call(["make", "-s", "-C", HERE, "liboracle.so"])
    return LIB


def lib():
    global _lib
    if _lib is None:
        if not os.path.exists(LIB):
            build()
        L = C.CDLL(LIB)
        L.oracle_libm_exp.restype = C.c_double
        L.oracle_libm_exp.argtypes = [C.c_double]
        L.oracle_confidence.restype = C.c_double
        L.oracle_confidence.argtypes = [_p, C.c_double, _p]
        L.oracle_features.restype = None
        L.oracle_features.argtypes = [C.POINTER(_Sent), C.POINTER(_Lex), C.c_int, C.c_int,
                                      C.c_double, C.c_double, _p]
        L.oracle_score_doc.restype = None
        L.oracle_score_doc.argtypes = [C.POINTER(_Sent), C.POINTER(_Lex), _p, C.c_double,
                                       C.c_int, C.c_int, C.c_int, C.c_int, _p]
        L.oracle_nw.restype = C.c_int
        L.oracle_nw.argtypes = [_p, C.c_int, C.c_int, C.c_double, _p, _p, _p, _p, _p]
        L.oracle_mine.restype = None
        L.oracle_mine.argtypes = [C.POINTER(_Sent), C.POINTER(_Docs), C.POINTER(_Lex), _p,
                                  C.c_double, C.c_double, C.c_double, _p, _p, _p, _p, C.c_int]
        L.oracle_tune.restype = None
        L.oracle_tune.argtypes = [C.POINTER(_Sent), C.POINTER(_Docs), C.POINTER(_Lex), _p,
                                  C.c_double, _p, C.c_int, _p, C.c_int, _p, _p, _p, _p, C.c_int]
        _lib = L
    return _lib


def _a(x, dt):
    return np.ascontiguousarray(np.asarray(x, dtype=dt))


class HostBatch:
    """Keeps the numpy arrays alive behind the C structs."""

    def __init__(self, corpus, plex, src0=None, n=None, tgt0=None, m=None):
        c = corpus
        self.keep = [
            _a(c.n_tok, np.int32), _a(c.n_punct, np.int32), _a(c.n_alpha, np.int32),
            _a(c.tok_off, np.int32), _a(c.tok_id, np.int32), _a(c.tok_alpha, np.uint32),
            _a(c.dig_off, np.int32), _a(c.dig_id, np.int32),
        ]
        self.sent = _Sent(c.n_sent, *[k.ctypes.data for k in self.keep])
        d = [_a(c.src0 if src0 is None else src0, np.int32), _a(c.n if n is None else n, np.int32),
             _a(c.tgt0 if tgt0 is None else tgt0, np.int32), _a(c.m if m is None else m, np.int32)]
        self.docs_arr = d
        self.docs = _Docs(len(d[1]), *[k.ctypes.data for k in d])
        lx = [_a(plex.fwd_off, np.int32), _a(plex.fwd_cand, np.int32),
              _a(plex.rev_off, np.int32), _a(plex.rev_cand, np.int32)]
        self.lx = lx
        self.lex = _Lex(plex.n_ids, *[k.ctypes.data for k in lx])


def _w(model) -> np.ndarray:
    w = [float(x) for x in list(model.weights)[:7]]
    return _a(w + [0.0] * (7 - len(w)), np.float64)


def libm_exp(x: float) -> float:
    return lib().oracle_libm_exp(float(x))


def score_doc(hb: HostBatch, model, d: int) -> np.ndarray:
    n, m = int(hb.docs_arr[1][d]), int(hb.docs_arr[3][d])
    out = np.empty((n, m), dtype=np.float64)
    w = _w(model)
    lib().oracle_score_doc(C.byref(hb.sent), C.byref(hb.lex), w.ctypes.data, float(model.bias),
                           int(hb.docs_arr[0][d]), n, int(hb.docs_arr[2][d]), m, out.ctypes.data)
    return out


def features(hb: HostBatch, s: int, t: int, ps: float, pt: float) -> np.ndarray:
    out = np.empty(7, dtype=np.float64)
    lib().oracle_features(C.byref(hb.sent), C.byref(hb.lex), s, t, ps, pt, out.ctypes.data)
    return out


def nw(S: np.ndarray, penalty: float):
    """(cost, ops, i, j) with moves in forward order (ops 0=D 1=GS 2=GT)."""
    S = _a(S, np.float64)
    n, m = S.shape
    op = np.empty(n + m, dtype=np.int8)
    mi = np.empty(n + m, dtype=np.int32)
    mj = np.empty(n + m, dtype=np.int32)
    cost = C.c_double()
    k = lib().oracle_nw(S.ctypes.data, n, m, float(penalty), C.byref(cost), op.ctypes.data,
                        mi.ctypes.data, mj.ctypes.data, None)
    return cost.value, op[:k].copy(), mi[:k].copy(), mj[:k].copy()


def mine(hb: HostBatch, model, threshold: float, penalty: float, threads: int = 1):
    n, m = hb.docs_arr[1], hb.docs_arr[3]
    cap = np.minimum(n, m).clip(min=0).astype(np.int64)
    off = np.zeros(len(n), dtype=np.int64)
    if len(n) > 1:
        off[1:] = np.cumsum(cap)[:-1]
    rec = np.zeros(max(int(cap.sum()), 1), dtype=RECORD)
    cnt = np.zeros(len(n), dtype=np.int32)
    cost = np.zeros(len(n), dtype=np.float64)
    w = _w(model)
    lib().oracle_mine(C.byref(hb.sent), C.byref(hb.docs), C.byref(hb.lex), w.ctypes.data,
                      float(model.bias), float(threshold), float(penalty), off.ctypes.data,
                      rec.ctypes.data, cnt.ctypes.data, cost.ctypes.data, int(threads))
    parts = [rec[off[d] : off[d] + cnt[d]] for d in range(len(n))]
    dense = np.concatenate(parts) if parts else np.zeros(0, dtype=RECORD)
    return dense, cost


def tune(hb: HostBatch, model, penalties, thresholds, gold_keys, threads: int = 1):
    pen = _a(penalties, np.float64)
    thr = _a(thresholds, np.float64)
    goff = np.zeros(len(gold_keys) + 1, dtype=np.int64)
    goff[1:] = np.cumsum([len(g) for g in gold_keys])
    gall = _a(np.concatenate([np.sort(np.asarray(g, np.int64)) for g in gold_keys])
              if gold_keys else np.zeros(0), np.int64)
    pred = np.zeros((len(pen), len(thr)), dtype=np.int64)
    hit = np.zeros_like(pred)
    w = _w(model)
    lib().oracle_tune(C.byref(hb.sent), C.byref(hb.docs), C.byref(hb.lex), w.ctypes.data,
                      float(model.bias), pen.ctypes.data, len(pen), thr.ctypes.data, len(thr),
                      gall.ctypes.data, goff.ctypes.data, pred.ctypes.data, hit.ctypes.data,
                      int(threads))
    return pred, hit
