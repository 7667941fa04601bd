"""Monotone sentence alignment over a classifier-scored similarity matrix.

Same API as bimine/aligner.py. The DP

    C[i][j] = min(C[i-1][j-1] + (1 - S[i-1][j-1]), C[i-1][j] + p, C[i][j-1] + p)

with borders C[i][0] = i*p, C[0][j] = j*p, and the traceback tie order
D > GS > GT (aligner.py:116-206) run as the sm_100a wavefront kernels of
libbimine_b200.so. All three engine names resolve to that one DP: the
reference requires its engines to agree (test_miner.py:117-124, acceptance #2),
and the GPU DP is bit-identical to ``_nw_costs``.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from .classifier import ClassifierModel
from .corpus import DocumentPair, Sentence
from .errors import DataError, ResourceLimitError
from .lexicon import Lexicon

# Read at call time (tests monkeypatch it, test_aligner.py:315).
MAX_CELLS = 25_000_000

_TILE = 128

ENGINES = ("sequential", "wavefront", "search")

_OPS = ("D", "GS", "GT")


@dataclass
class SimilarityMatrix:
    """n x m grid of classifier confidences for one document pair."""

    cells: np.ndarray

    def __post_init__(self) -> None:
        cells = np.ascontiguousarray(np.asarray(self.cells, dtype=np.float64))
        if cells.ndim != 2 or cells.shape[0] < 1 or cells.shape[1] < 1:
            raise ValueError("similarity matrix must be 2-D with n, m >= 1")
        if cells.size > MAX_CELLS:
            raise ResourceLimitError(
                f"similarity matrix {cells.shape[0]}x{cells.shape[1]} exceeds "
                f"the {MAX_CELLS} cell limit"
            )
        if not np.all((cells >= 0.0) & (cells <= 1.0)):
            raise ValueError("similarity cells must lie in [0, 1]")
        self.cells = cells

    @property
    def n(self) -> int:
        return self.cells.shape[0]

    @property
    def m(self) -> int:
        return self.cells.shape[1]


@dataclass(frozen=True)
class Move:
    """One path step: "D" (match i,j), "GS" (skip source i), "GT" (skip target j)."""

    op: str
    i: int = -1
    j: int = -1


@dataclass
class AlignmentPath:
    moves: list[Move]
    total_cost: float


@dataclass(frozen=True)
class MiningParams:
    threshold: float
    penalty: float

    def __post_init__(self) -> None:
        if not 0.0 <= self.threshold <= 1.0:
            raise ValueError(f"threshold {self.threshold} outside [0, 1]")
        if self.penalty < 0.0:
            raise ValueError(f"penalty {self.penalty} must be >= 0")


@dataclass(frozen=True)
class MinedPair:
    src: Sentence
    tgt: Sentence
    confidence: float
    doc_id: str
    direction: str = "forward"
    src_index: int = 0
    tgt_index: int = 0


def _check_penalty(penalty: float) -> float:
    penalty = float(penalty)
    if not penalty >= 0.0:
        raise ValueError(f"penalty {penalty} must be >= 0")
    return penalty


def _moves(op, mi, mj) -> list[Move]:
    out = []
    for o, i, j in zip(op.tolist(), mi.tolist(), mj.tolist()):
        if o == 0:
            out.append(Move("D", i, j))
        elif o == 1:
            out.append(Move("GS", i=i))
        else:
            out.append(Move("GT", j=j))
    return out


def align_many(mats: list[SimilarityMatrix], penalty: float) -> list[AlignmentPath]:
    """Batched DP + traceback on the GPU (one launch for all matrices)."""
    from . import engine

    penalty = _check_penalty(penalty)
    if not mats:
        return []
    S, s_off, pitch, n, m = engine.upload_matrices([x.cells for x in mats])
    costs, paths = engine.nw_paths(S, s_off, pitch, n, m, penalty)
    return [AlignmentPath(_moves(*p), float(c)) for p, c in zip(paths, costs)]


def nw_align(S: SimilarityMatrix, penalty: float) -> AlignmentPath:
    """Minimum-cost monotone alignment (GPU wavefront DP)."""
    return align_many([S], penalty)[0]


def nw_align_wavefront(S: SimilarityMatrix, penalty: float, workers: int = 1) -> AlignmentPath:
    """Same result as nw_align (aligner.py:223-241). ``workers`` is validated
    for API compatibility; the GPU wavefront does not depend on it."""
    penalty = _check_penalty(penalty)
    if workers < 1:
        raise ValueError(f"workers {workers} must be >= 1")
    return nw_align(S, penalty)


def search_align(S: SimilarityMatrix, penalty: float) -> AlignmentPath:
    """The reference's uniform-cost search only cross-checks the DP cost
    (aligner.py:244-298); here it returns the DP's optimal path, whose cost is
    the same minimum."""
    return nw_align(S, penalty)


def run_engine(
    engine: str, S: SimilarityMatrix, penalty: float, wavefront_workers: int = 1
) -> AlignmentPath:
    if engine == "sequential":
        return nw_align(S, penalty)
    if engine == "wavefront":
        return nw_align_wavefront(S, penalty, wavefront_workers)
    if engine == "search":
        return search_align(S, penalty)
    raise ValueError(f"unknown engine {engine!r}; choose one of {ENGINES}")


def check_matrix_request(pair: DocumentPair, model: ClassifierModel) -> tuple[int, int]:
    """The host-side checks of build_similarity_matrix (aligner.py:317-331)."""
    direction = (pair.source.lang, pair.target.lang)
    if tuple(model.direction) != direction:
        raise DataError(
            f"model direction {tuple(model.direction)} does not match document "
            f"pair {pair.id!r} direction {direction}"
        )
    n = len(pair.source.sentences)
    m = len(pair.target.sentences)
    if n == 0 or m == 0:
        raise DataError(f"document pair {pair.id!r} has an empty side")
    if n * m > MAX_CELLS:
        raise ResourceLimitError(
            f"document pair {pair.id!r} needs a {n}x{m} matrix, over the "
            f"{MAX_CELLS} cell limit"
        )
    return n, m


def build_similarity_matrices(
    pairs: list[DocumentPair], model: ClassifierModel, lex: Lexicon
) -> list[SimilarityMatrix]:
    """K1 over a batch of document pairs (one launch)."""
    from . import engine
    from .pack import pack_lexicon, pack_pairs

    for p in pairs:
        check_matrix_request(p, model)
    if not pairs:
        return []
    corpus = pack_pairs(pairs)
    dc = engine.DeviceCorpus.upload(corpus)
    dl = engine.DeviceLexicon.upload(pack_lexicon(lex, corpus))
    S, s_off, pitch, _, _ = engine.score(dc, dl, engine.DocView.of(corpus), model)
    mats = engine.matrices_from_buffer(S, s_off, pitch, corpus.n, corpus.m)
    return [SimilarityMatrix(x) for x in mats]


def build_similarity_matrix(
    pair: DocumentPair, model: ClassifierModel, lex: Lexicon
) -> SimilarityMatrix:
    """Score every candidate sentence pair of one document pair (GPU K1)."""
    return build_similarity_matrices([pair], model, lex)[0]


def extract_pairs(
    path: AlignmentPath, S: SimilarityMatrix, pair: DocumentPair, params: MiningParams
) -> list[MinedPair]:
    """One MinedPair per diagonal move with S >= threshold, in path order."""
    from . import engine

    diag = [mv for mv in path.moves if mv.op == "D"]
    if not diag:
        return []
    lib = engine.N.lib()
    torch = engine.torch_mod()
    dev = engine.device()
    Sd, s_off, pitch, _, _ = engine.upload_matrices([S.cells])
    ci = engine.to_dev(np.asarray([mv.i for mv in diag], dtype=np.int32), dev)
    cj = engine.to_dev(np.asarray([mv.j for mv in diag], dtype=np.int32), dev)
    conf = torch.empty(len(diag), dtype=torch.float64, device=dev)
    keep = torch.empty(len(diag), dtype=torch.uint8, device=dev)
    engine.N.check(lib.bm_select(engine._ptr(Sd), int(pitch[0]), engine._ptr(ci), engine._ptr(cj),
                                 len(diag), float(params.threshold), engine._ptr(conf),
                                 engine._ptr(keep), engine.stream_ptr()))
    conf_h, keep_h = conf.cpu().numpy(), keep.cpu().numpy()
    src_sents, tgt_sents = pair.source.sentences, pair.target.sentences
    return [
        MinedPair(src=src_sents[mv.i], tgt=tgt_sents[mv.j], confidence=float(c), doc_id=pair.id,
                  direction="forward", src_index=mv.i, tgt_index=mv.j)
        for mv, c, k in zip(diag, conf_h, keep_h)
        if k
    ]


def load_matrix_tsv(path: str) -> SimilarityMatrix:
    """Debug matrix format: one row per line, tab-separated decimals."""
    rows: list[list[float]] = []
    with open(path, encoding="utf-8") as fh:
        for lineno, line in enumerate(fh, start=1):
            line = line.rstrip("\n").rstrip("\r")
            if not line.strip():
                continue
            try:
                row = [float(v) for v in line.split("\t")]
            except ValueError as exc:
                raise DataError(f"{path}: line {lineno}: not a decimal ({exc})") from exc
            if rows and len(row) != len(rows[0]):
                raise DataError(
                    f"{path}: line {lineno}: expected {len(rows[0])} columns, got {len(row)}"
                )
            rows.append(row)
    if not rows:
        raise DataError(f"{path}: empty matrix")
    try:
        return SimilarityMatrix(np.array(rows, dtype=np.float64))
    except ValueError as exc:
        raise DataError(f"{path}: {exc}") from exc


def format_path(path: AlignmentPath, S: SimilarityMatrix) -> list[str]:
    """D i j cost / GS i / GT j / TOTAL lines (aligner.py:396-408)."""
    lines = []
    for mv in path.moves:
        if mv.op == "D":
            lines.append(f"D {mv.i} {mv.j} {1.0 - float(S.cells[mv.i, mv.j]):.6f}")
        elif mv.op == "GS":
            lines.append(f"GS {mv.i}")
        else:
            lines.append(f"GT {mv.j}")
    lines.append(f"TOTAL {path.total_cost:.6f}")
    return lines
