"""Translation-pair classifier: model type, model JSON, features, confidence.

Mirrors bimine/classifier.py: constants (:23-33), ``FeatureVector`` /
``ClassifierModel`` (:36-49), ``extract_features`` (:68-97), ``confidence``
(:107-117) and the model file format (:235-287). Feature extraction and the
sigmoid run in the scoring kernels (bm_features / bm_confidence); training
(:145-232) is not part of the B200 hot path -- train once with the reference
and load the JSON.
"""

from __future__ import annotations

import json
from dataclasses import dataclass

import numpy as np

from .corpus import Sentence
from .errors import DataError

SCHEMA_ID = "pairwise-v1"
FEATURE_COUNT = 7
MODEL_VERSION = 1

_P_MIN = 1e-300
_P_MAX = 1.0 - 2.0**-53

THRESHOLD_GRID = tuple(round(0.05 * k, 2) for k in range(1, 20))
DEFAULT_PENALTY = 0.2


@dataclass
class FeatureVector:
    values: list[float]
    schema_id: str = SCHEMA_ID


@dataclass
class ClassifierModel:
    schema_id: str
    weights: list[float]
    bias: float
    direction: tuple[str, str]
    default_threshold: float
    default_penalty: float
    version: int = MODEL_VERSION
    trained_on: dict | None = None


def _features_batch(items, lex) -> np.ndarray:
    """[(src Sentence, tgt Sentence, src_pos, tgt_pos)] -> float64 [k, 7] on the GPU."""
    from . import engine
    from .pack import Packer, pack_lexicon

    pk = Packer()
    qs, qt, ps, pt = [], [], [], []
    for src, tgt, sp, tp in items:
        a, b = pk.add_sentence_pair(src, tgt)
        qs.append(a)
        qt.append(b)
        ps.append(float(sp))
        pt.append(float(tp))
    corpus = pk.finish()
    dc = engine.DeviceCorpus.upload(corpus)
    dl = engine.DeviceLexicon.upload(pack_lexicon(lex, corpus))
    return engine.features(dc, dl, qs, qt, ps, pt)


def extract_features(
    src: Sentence, tgt: Sentence, src_pos: float, tgt_pos: float, lex
) -> FeatureVector:
    """The 7-feature vector of one candidate pair (computed by bm_features)."""
    vals = _features_batch([(src, tgt, src_pos, tgt_pos)], lex)[0]
    return FeatureVector(values=[float(v) for v in vals])


def confidence(model: ClassifierModel, f: FeatureVector) -> float:
    """sigmoid(w . f + b) clamped to [1e-300, 1 - 2^-53] (bm_confidence)."""
    if f.schema_id != model.schema_id:
        raise DataError(
            f"feature schema {f.schema_id!r} does not match model schema "
            f"{model.schema_id!r}"
        )
    from . import engine

    vals = [float(v) for v in f.values][:FEATURE_COUNT]
    # zip(weights, values) in the reference: missing values contribute nothing
    vals += [0.0] * (FEATURE_COUNT - len(vals))
    n_used = min(len(f.values), len(model.weights))
    weights = list(model.weights)[:n_used]
    m = ClassifierModel(model.schema_id, weights, model.bias, model.direction,
                        model.default_threshold, model.default_penalty)
    return float(engine.confidences(np.asarray([vals], dtype=np.float64), m)[0])


def train(*_args, **_kwargs):
    raise NotImplementedError(
        "classifier training is not part of the B200 hot path; train with the "
        "reference package (bimine.classifier.train) and load the saved JSON"
    )


def model_to_json(model: ClassifierModel) -> str:
    payload = {
        "version": model.version,
        "schema_id": model.schema_id,
        "direction": list(model.direction),
        "weights": model.weights,
        "bias": model.bias,
        "default_threshold": model.default_threshold,
        "default_penalty": model.default_penalty,
        "trained_on": model.trained_on,
    }
    return json.dumps(payload, sort_keys=True, indent=2) + "\n"


def save_model(model: ClassifierModel, path: str) -> None:
    with open(path, "w", encoding="utf-8") as fh:
        fh.write(model_to_json(model))


def load_model(path: str) -> ClassifierModel:
    """Read a model JSON with the reference's validation (classifier.py:254-287)."""
    try:
        with open(path, encoding="utf-8") as fh:
            payload = json.load(fh)
    except json.JSONDecodeError as exc:
        raise DataError(f"{path}: not a valid model file ({exc.msg})") from exc
    if not isinstance(payload, dict) or "version" not in payload:
        raise DataError(f"{path}: not a valid model file (no version)")
    if payload["version"] != MODEL_VERSION:
        raise DataError(
            f"{path}: unsupported model version {payload['version']!r} (expected {MODEL_VERSION})"
        )
    try:
        model = ClassifierModel(
            schema_id=payload["schema_id"],
            weights=[float(w) for w in payload["weights"]],
            bias=float(payload["bias"]),
            direction=(payload["direction"][0], payload["direction"][1]),
            default_threshold=float(payload["default_threshold"]),
            default_penalty=float(payload["default_penalty"]),
            version=payload["version"],
            trained_on=payload.get("trained_on"),
        )
    except (KeyError, IndexError, TypeError, ValueError) as exc:
        raise DataError(f"{path}: malformed model file ({exc})") from exc
    if len(model.weights) != FEATURE_COUNT:
        raise DataError(
            f"{path}: model has {len(model.weights)} weights; schema "
            f"{model.schema_id!r} requires {FEATURE_COUNT}"
        )
    if not (0.0 <= model.default_threshold <= 1.0) or model.default_penalty < 0:
        raise DataError(f"{path}: default parameters out of range")
    return model
