"""Error hierarchy of the drop-in (mirrors bimine/errors.py:4-16).

``DataError`` maps to CLI exit code 2 in the reference; ``ResourceLimitError``
is raised when a similarity matrix would exceed ``aligner.MAX_CELLS`` and is
caught per document by the miner (bimine/miner.py:179-180).
"""


class BimineError(Exception):
    """Root of every error raised by this package."""


class DataError(BimineError):
    """Bad input: malformed files, out-of-range values, direction mismatches."""


class ResourceLimitError(DataError):
    """An input is over a hard size bound (similarity-matrix cell cap)."""


class NativeUnavailableError(BimineError, RuntimeError):
    """The sm_100a library is missing or no CUDA device is usable.

    There is deliberately no CPU fallback: every hot-path entry point raises
    this instead of silently computing on the host.
    """
