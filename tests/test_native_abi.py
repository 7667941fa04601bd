"""The C-ABI library builds, loads without a GPU and exports every symbol of
include/bimine_b200.h; without a device the hot path fails loudly."""

import ctypes
import os
import re

import numpy as np
import pytest

import paper_1509_08639_b200 as bm
from conftest import ROOT, have_gpu
from paper_1509_08639_b200 import _native

HEADER = os.path.join(ROOT, "include", "bimine_b200.h")


def declared_symbols(header=HEADER):
    text = open(header).read()
    return sorted(set(re.findall(r"^\s*(?:[\w\s\*]+?)\b(bm_\w+)\s*\(", text, flags=re.M)))


@pytest.fixture(scope="module")
def lib():
    from paper_1509_08639_b200 import _build

    _build.build()
    return _native.load_library()


def test_header_declares_the_entry_points():
    syms = declared_symbols()
    for name in ("bm_score", "bm_nw", "bm_traceback", "bm_extract", "bm_mine", "bm_mine_host",
                 "bm_tune", "bm_compact", "bm_features", "bm_confidence", "bm_select"):
        assert name in syms


def test_library_exports_every_declared_symbol(lib):
    for name in declared_symbols():
        assert hasattr(lib, name), name
    assert set(declared_symbols()) == set(_native.EXPORTED)
    synth_h = os.path.join(ROOT, "include", "bimine_synth.h")
    for name in declared_symbols(synth_h):
        assert hasattr(lib, name), name
    assert set(declared_symbols(synth_h)) == set(_native.SYNTH_SIGS)


def test_abi_version_and_record_layout(lib):
    assert lib.bm_abi_version() == 2
    assert ctypes.sizeof(_native.Record) == 24
    assert np.dtype(_native.RECORD_DTYPE).itemsize == 24
    assert lib.bm_dirs_words(128, 4) == 32
    assert lib.bm_dirs_words(129, 5) == 2 * 2 * 32


def test_sm100a_code_in_library():
    path = _native.LIB_PATH
    data = open(path, "rb").read()
    assert b"sm_100a" in data or b"sm_100" in data


@pytest.mark.skipif(have_gpu(), reason="checks the no-GPU behaviour")
def test_no_cpu_fallback_without_device(world500):
    lex, fwd, _ = world500
    from conftest import load_docs, pairs_of

    pair = pairs_of(load_docs("docs40.jsonl"))[0]
    with pytest.raises(bm.NativeUnavailableError):
        bm.build_similarity_matrix(pair, fwd, lex)
    with pytest.raises(bm.NativeUnavailableError):
        bm.nw_align(bm.SimilarityMatrix(np.eye(2)), 0.5)
    cfg = bm.MinerConfig(bm.MiningParams(0.5, 0.2))
    with pytest.raises(bm.NativeUnavailableError):
        bm.mine_document(pair, fwd, lex, cfg)
