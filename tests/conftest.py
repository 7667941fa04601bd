import gzip
import json
import os
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
GOLDEN = os.path.join(ROOT, "tests", "golden")
sys.path.insert(0, ROOT)

import paper_1509_08639_b200 as bm  # noqa: E402


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200) and the built library")
    config.addinivalue_line("markers", "slow: long-running")


def golden(name: str) -> str:
    return os.path.join(GOLDEN, name)


def load_docs(name: str) -> list[dict]:
    path = golden(name)
    opener = gzip.open if name.endswith(".gz") else open
    with opener(path, "rt", encoding="utf-8") as fh:
        return [json.loads(line) for line in fh if line.strip()]


def pairs_of(docs: list[dict]):
    return [bm.parse_document_pair(d, "mem", i) for i, d in enumerate(docs, 1)]


def stacked(name: str) -> list[np.ndarray]:
    z = np.load(golden(name))
    out, o = [], 0
    for n, m in z["shape"]:
        out.append(z["flat"][o : o + n * m].reshape(n, m))
        o += n * m
    return out


def dp_cases(name: str):
    z = np.load(golden(name))
    out = []
    for k in range(len(z["cost"])):
        out.append((tuple(z["shape"][k]), float(z["cost"][k]), z["ops"][z["off"][k] : z["off"][k + 1]]))
    return out


def moves_from_ops(ops):
    i = j = 0
    out = []
    for o in ops.tolist():
        if o == 0:
            out.append(bm.Move("D", i, j))
            i += 1
            j += 1
        elif o == 1:
            out.append(bm.Move("GS", i=i))
            i += 1
        else:
            out.append(bm.Move("GT", j=j))
            j += 1
    return out


def stress_lexicon():
    d = json.load(open(golden("lex_stress.json")))
    return bm.Lexicon(direction=tuple(d["direction"]),
                      entries={k: [tuple(c) for c in v] for k, v in d["entries"].items()})


@pytest.fixture(scope="session")
def world500():
    lex = bm.load_lexicon(golden("lex500.tsv"), "xx", "yy")
    fwd = bm.load_model(golden("model500_fwd.json"))
    bwd = bm.load_model(golden("model500_bwd.json"))
    return lex, fwd, bwd


@pytest.fixture(scope="session")
def world5k():
    lex = bm.load_lexicon(golden("lex5k.tsv"), "xx", "yy")
    fwd = bm.load_model(golden("model5k_fwd.json"))
    bwd = bm.load_model(golden("model5k_bwd.json"))
    return lex, fwd, bwd


@pytest.fixture(scope="session")
def oracle_mod():
    sys.path.insert(0, os.path.join(ROOT, "oracle"))
    import oracle  # test infrastructure

    oracle.build()
    return oracle


def have_gpu() -> bool:
    try:
        from paper_1509_08639_b200 import _native

        return _native.load_library().bm_device_count() > 0
    except Exception:
        return False
