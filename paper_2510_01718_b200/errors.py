"""Exception types of the drop-in API (ref: pkg/src/bdattn/errors.py:4-9).

Same names and the same ``ValueError`` base as the reference, so callers'
``except ShapeError`` / ``except ValueError`` clauses keep working.
"""


class ShapeError(ValueError):
    """Operand shapes are incompatible with the requested operation."""


class PrecisionError(ValueError):
    """Operands carry different element precisions."""


class NativeLibraryError(RuntimeError):
    """The CUDA extension is missing, failed to load, or a CUDA call failed.

    There is no CPU fallback: the product path fails loudly instead.
    """
