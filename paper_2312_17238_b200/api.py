"""The public value types of the hot path, taken from the reference package.

The reference package ``moe_offload`` stays in place (BASELINE north_star): this
engine is a drop-in backend behind its API, so it returns the reference's own
objects -- ``StoreEvent``/``ExpertKey``/``CacheConfig`` (store.py:35-73),
``recall`` and the event JSONL codec (store.py:223-265), ``Trace``/
``TraceRecord``/``config_digest`` (trace.py:33-105), ``SpeculationConfig``/
``GenerationResult`` (engine.py:43-94), the samplers (model.py:374-401) -- and
the reference's analysis tools (``replay``, ``guess_recall``, ``recall``) and
equality checks (``replay(...).events == eng.events``) work on its output
unchanged.

``moe_offload`` is imported from the environment, else from the reference
install under ``<repo>/baseline/_ref`` (``pip install --target baseline/_ref``).
"""

from __future__ import annotations

import os
import sys

try:
    import moe_offload  # noqa: F401
except ImportError:  # the in-repo reference install
    _ref = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))),
                        "baseline", "_ref")
    if os.path.isdir(os.path.join(_ref, "moe_offload")):
        sys.path.append(_ref)
    try:
        import moe_offload  # noqa: F401
    except ImportError as exc:  # pragma: no cover
        raise ImportError(
            "paper_2312_17238_b200 is a backend of the reference package moe_offload: "
            "install it (pip install <reference>/pkg, or --target baseline/_ref)") from exc

from moe_offload.engine import GenerationResult, SpeculationConfig  # noqa: E402,F401
from moe_offload.model import NonFiniteError, make_sampler, sample_greedy  # noqa: E402,F401
from moe_offload.quant import QuantFormatError  # noqa: E402,F401
from moe_offload.store import (ACQUIRE_KINDS, EVENT_KINDS, LOAD_KINDS,  # noqa: E402,F401
                               CacheConfig, ExpertKey, StoreEvent, UnknownExpertError,
                               events_from_jsonl, events_to_jsonl, recall)
from moe_offload.trace import (Trace, TraceFormatError, TraceRecord,  # noqa: E402,F401
                               config_digest)
