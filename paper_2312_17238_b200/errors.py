"""The reference's exception classes (model.py:36-37, store.py:42-43,
quant.py:30-31, trace.py:29-30), re-exported so that callers catching the
reference's exceptions catch the engine's."""

from .api import NonFiniteError, QuantFormatError, TraceFormatError, UnknownExpertError  # noqa: F401
