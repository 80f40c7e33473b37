"""Exception classes of the reference API (same names, same base classes)."""


class NonFiniteError(ValueError):
    """A hidden state or logit stopped being finite (reference model.py:36-37)."""


class UnknownExpertError(KeyError):
    """Requested key is outside the store's expert table (reference store.py:42-43)."""


class QuantFormatError(ValueError):
    """Corrupted or inconsistent quantized block (reference quant.py:30-31)."""


class TraceFormatError(ValueError):
    """Malformed or inconsistent trace data (reference trace.py:29-30)."""
