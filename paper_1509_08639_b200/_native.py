"""ctypes binding of libbimine_b200.so (include/bimine_b200.h).

The library is the only compute path: if it is missing, fails to load, or no
CUDA device is visible, every hot-path call raises NativeUnavailableError.
There is no CPU fallback anywhere in the package.
"""

from __future__ import annotations

import ctypes as C
import os
import threading

from .errors import NativeUnavailableError, ResourceLimitError

# BM_LIB_PATH: load an instrumented variant (tools/nw_trace.py); default in-tree
LIB_PATH = os.environ.get("BM_LIB_PATH") or os.path.join(os.path.dirname(os.path.abspath(__file__)),
                                                        "libbimine_b200.so")

BM_OK, BM_EINVAL, BM_ECUDA, BM_ENOMEM, BM_ELIMIT, BM_EUNSUPPORTED = 0, -1, -2, -3, -4, -5
MOVE_D, MOVE_GS, MOVE_GT = 0, 1, 2

_p = C.c_void_p
_i32p = C.POINTER(C.c_int32)


class Sentences(C.Structure):
    _fields_ = [
        ("n_sent", C.c_int32),
        ("n_tok", _p), ("n_punct", _p), ("n_alpha", _p),
        ("tok_off", _p), ("tok_id", _p), ("tok_alpha", _p),
        ("dig_off", _p), ("dig_id", _p),
    ]


class Wire(C.Structure):
    _fields_ = [
        ("n_sent", C.c_int32),
        ("n_tok", _p), ("n_punct", _p), ("n_alpha", _p),
        ("tok_off", _p), ("tok_id", _p), ("tok_alpha", _p),
        ("dig_off", _p), ("dig_id", _p),
    ]


class WirePacked(C.Structure):
    _fields_ = [
        ("n_sent", C.c_int32),
        ("tok_off", _p), ("dig_off", _p), ("counts", _p), ("tok_off32", _p),
        ("dig_off32", _p), ("tok_pk", _p), ("dig_id", _p),
    ]


class Docs(C.Structure):
    _fields_ = [("n_docs", C.c_int32), ("src0", _p), ("n", _p), ("tgt0", _p), ("m", _p)]


class LexiconC(C.Structure):
    _fields_ = [("n_ids", C.c_int32), ("fwd_off", _p), ("fwd_cand", _p),
                ("rev_off", _p), ("rev_cand", _p)]


class ModelC(C.Structure):
    _fields_ = [("w", C.c_double * 7), ("bias", C.c_double)]


class Record(C.Structure):
    _fields_ = [("doc", C.c_int32), ("i", C.c_int32), ("j", C.c_int32),
                ("pad", C.c_int32), ("conf", C.c_double)]


RECORD_DTYPE = [("doc", "<i4"), ("i", "<i4"), ("j", "<i4"), ("pad", "<i4"), ("conf", "<f8")]

class IngestArrays(C.Structure):
    _fields_ = [("n_sent", C.c_int32), ("n_docs", C.c_int32), ("n_ids", C.c_int32),
                ("n_skipped", C.c_int32), ("n_tok_entries", C.c_int64),
                ("n_dig_entries", C.c_int64)] + [
        (name, C.c_void_p) for name in ("n_tok", "n_punct", "n_alpha", "tok_off", "tok_id",
                                        "tok_alpha", "dig_off", "dig_id", "src0", "n", "tgt0",
                                        "m")]


_SIGS = {
    "bm_abi_version": (C.c_int, []),
    "bm_trim": (C.c_int, []),
    "bm_last_error": (C.c_char_p, []),
    "bm_device_count": (C.c_int, []),
    "bm_dirs_words": (C.c_int64, [C.c_int32, C.c_int32]),
    "bm_launches": (C.c_int64, []),
    "bm_probe_fp64": (C.c_int, [_p, C.c_int32, C.c_int32, _p]),
    "bm_score": (C.c_int, [C.POINTER(Sentences), C.POINTER(Docs), _p, _p, C.POINTER(LexiconC),
                           C.POINTER(ModelC), _p, _p, _p, _p]),
    "bm_features": (C.c_int, [C.POINTER(Sentences), C.POINTER(LexiconC), _p, _p, _p, _p,
                              C.c_int32, _p, _p]),
    "bm_confidence": (C.c_int, [_p, C.c_int32, C.POINTER(ModelC), _p, _p]),
    "bm_nw": (C.c_int, [_p, _p, _p, _p, _p, _p, _p, C.c_int32, C.c_double, _p, _p, _p, _p]),
    "bm_traceback": (C.c_int, [_p, _p, _p, _p, C.c_int32, _p, _p, _p, _p, _p, _p]),
    "bm_extract": (C.c_int, [_p, _p, _p, _p, _p, _p, _p, C.c_int32, C.c_double, _p, _p, _p, _p]),
    "bm_select": (C.c_int, [_p, C.c_int64, _p, _p, C.c_int32, C.c_double, _p, _p, _p]),
    "bm_mine": (C.c_int, [C.POINTER(Sentences), C.POINTER(Docs), _p, _p, _p,
                          C.POINTER(LexiconC), C.POINTER(ModelC), C.c_double, C.c_double,
                          _p, _p, _p, _p, _p]),
    "bm_mine_host": (C.c_int, [C.POINTER(Sentences), C.POINTER(Docs), C.POINTER(LexiconC),
                               C.POINTER(ModelC), C.c_double, C.c_double, _p, C.c_int64,
                               C.POINTER(C.c_int64), _p, _p]),
    "bm_mine_host_wire": (C.c_int, [C.POINTER(Wire), C.POINTER(Docs), C.POINTER(LexiconC),
                                    C.POINTER(ModelC), C.c_double, C.c_double, _p, C.c_int64,
                                    C.POINTER(C.c_int64), _p, _p]),
    "bm_mine_host_packed": (C.c_int, [C.POINTER(WirePacked), C.POINTER(Docs), C.POINTER(LexiconC),
                                      C.POINTER(ModelC), C.c_double, C.c_double, _p, C.c_int64,
                                      C.POINTER(C.c_int64), _p, _p]),
    "bm_tune": (C.c_int, [C.POINTER(Sentences), C.POINTER(Docs), _p, _p, C.POINTER(LexiconC),
                          C.POINTER(ModelC), _p, C.c_int32, _p, C.c_int32, _p, _p, _p, _p,
                          C.c_int32, _p]),
    "bm_compact": (C.c_int, [_p, _p, _p, C.c_int32, _p, _p, _p]),
    "bm_merge_shards": (C.c_int, [_p, C.c_int64, _p, C.c_int32, C.c_int32, _p, _p, _p]),
    "bm_merge_bidir": (C.c_int, [_p, C.c_int64, _p, C.c_int64, C.c_int32, _p, _p, _p, _p, _p, _p,
                                 _p, _p]),
    "bm_ingest_jsonl": (C.c_int, [C.c_char_p, C.POINTER(C.c_void_p), C.c_char_p, C.c_int32]),
    "bm_ingest_free": (None, [C.c_void_p]),
    "bm_ingest_gold_jsonl": (C.c_int, [C.c_char_p, C.POINTER(C.c_void_p), C.c_char_p, C.c_int32]),
    "bm_ingest_gold": (C.c_int, [C.c_void_p, C.POINTER(C.c_void_p), C.POINTER(C.c_void_p),
                                 C.POINTER(C.c_int64)]),
    "bm_ingest_view": (C.c_int, [C.c_void_p, C.POINTER(IngestArrays)]),
    "bm_ingest_doc": (C.c_int, [C.c_void_p, C.c_int32, C.POINTER(C.c_char_p),
                                C.POINTER(C.c_char_p), C.POINTER(C.c_char_p)]),
    "bm_ingest_skipped": (C.c_int, [C.c_void_p, C.c_int32, C.POINTER(C.c_int64),
                                    C.POINTER(C.c_char_p), C.POINTER(C.c_char_p)]),
    "bm_ingest_lexicon": (C.c_int, [C.c_void_p, C.POINTER(C.c_char_p), C.POINTER(C.c_char_p),
                                    C.c_int64, C.POINTER(LexiconC)]),
    "bm_ingest_emit": (C.c_int, [C.c_void_p, _p, C.c_int64, _p, C.c_int64, C.c_int32, _p, _p, _p,
                                 C.POINTER(C.c_char_p), C.POINTER(C.c_int64), _p]),
    "bm_ingest_emit_merged": (C.c_int, [C.c_void_p, _p, C.c_int64, _p, C.POINTER(C.c_char_p),
                                        C.POINTER(C.c_int64), _p]),
    "bm_ingest_norm_keys": (C.c_int, [C.c_void_p, C.POINTER(C.c_void_p)]),
    "bm_ingest_jsonl_range": (C.c_int, [C.c_char_p, C.c_int64, C.c_int64, C.c_int64,
                                        C.POINTER(C.c_void_p), C.POINTER(C.c_int64), C.c_char_p,
                                        C.c_int32]),
    "bm_ingest_seen": (C.c_int, [C.c_void_p, C.c_int32, C.POINTER(C.c_void_p),
                                 C.POINTER(C.c_int64)]),
}

EXPORTED = tuple(_SIGS)


class SynthSpec(C.Structure):
    _fields_ = [("vocab", C.c_int32), ("noise", C.c_double), ("digit_rate", C.c_double),
                ("seed", C.c_uint64)]


class SynthArrays(C.Structure):
    _fields_ = [(k, C.c_int64) for k in ("n_sent", "n_docs", "n_tok_entries", "n_dig_entries",
                                          "n_gold")] + [
        (name, C.c_void_p) for name in ("n_tok", "n_punct", "n_alpha", "tok_off", "tok_id",
                                        "tok_alpha", "dig_off", "dig_id", "src0", "n", "tgt0",
                                        "m", "gold_off", "gold_i", "gold_j")]


# include/bimine_synth.h: benchmark input generation (not the mining boundary)
SYNTH_SIGS = {
    "bm_synth_generate": (C.c_int, [C.POINTER(SynthSpec), _p, _p, _p, _p, C.c_int64, C.c_int32,
                                    C.POINTER(C.c_void_p)]),
    "bm_synth_view": (C.c_int, [C.c_void_p, C.POINTER(SynthArrays)]),
    "bm_synth_free": (None, [C.c_void_p]),
    "bm_synth_jsonl": (C.c_int, [C.POINTER(SynthSpec), _p, _p, _p, _p, C.c_int64, C.c_int32,
                                 C.c_char_p]),
}

_lock = threading.Lock()
_lib: C.CDLL | None = None


def load_library(require_device: bool = False) -> C.CDLL:
    """Load the library (no GPU needed just to load and inspect it)."""
    global _lib
    with _lock:
        if _lib is None:
            if not os.path.exists(LIB_PATH):
                raise NativeUnavailableError(
                    f"{LIB_PATH} is missing; build it with "
                    "`python -c 'import __graft_entry__ as g; g.build()'`"
                )
            lib = C.CDLL(LIB_PATH)
            for name, (res, args) in {**_SIGS, **SYNTH_SIGS}.items():
                fn = getattr(lib, name)
                fn.restype = res
                fn.argtypes = args
            _lib = lib
    if require_device and _lib.bm_device_count() < 1:
        raise NativeUnavailableError("no CUDA device visible: the B200 kernels cannot run")
    return _lib


def lib() -> C.CDLL:
    """The library, with a usable CUDA device (hot-path entry)."""
    return load_library(require_device=True)


def check(rc: int) -> None:
    if rc == BM_OK:
        return
    msg = (load_library().bm_last_error() or b"").decode("utf-8", "replace")
    if rc == BM_EINVAL:
        raise ValueError(msg)
    if rc == BM_ELIMIT:
        raise ResourceLimitError(msg)
    if rc == BM_ENOMEM:
        raise MemoryError(msg)
    raise RuntimeError(f"libbimine_b200 error {rc}: {msg}")


def model_struct(model) -> ModelC:
    # confidence() zips weights with the 7 features (classifier.py:114-116):
    # extra weights are ignored, missing ones contribute nothing (z + 0.0 == z
    # for every z the sigmoid can tell apart), so pad/truncate to 7.
    m = ModelC()
    w = [float(x) for x in list(model.weights)[:7]]
    w += [0.0] * (7 - len(w))
    for k in range(7):
        m.w[k] = w[k]
    m.bias = float(model.bias)
    return m
