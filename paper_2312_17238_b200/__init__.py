"""B200-native decode-time MoE offloading engine (arXiv 2312.17238 hot path).

Drop-in for the reference ``moe_offload.engine.OffloadEngine``; the compute and
the expert store run in ``libmoeb200.so`` (CUDA, sm_100a) behind the C ABI of
``include/moeb200.h``.
"""

from .api import (ACQUIRE_KINDS, EVENT_KINDS, CacheConfig, ExpertKey, GenerationResult,
                  SpeculationConfig, StoreEvent, Trace, TraceRecord, events_from_jsonl,
                  events_to_jsonl, recall)
from .engine import DenseRunner, OffloadEngine, payload_nbytes, synthetic_model
from .errors import NonFiniteError, QuantFormatError, TraceFormatError, UnknownExpertError

__all__ = ["OffloadEngine", "DenseRunner", "CacheConfig", "SpeculationConfig", "ExpertKey", "StoreEvent",
           "Trace", "TraceRecord", "GenerationResult", "recall", "events_to_jsonl",
           "events_from_jsonl", "payload_nbytes", "synthetic_model", "NonFiniteError",
           "UnknownExpertError", "QuantFormatError", "TraceFormatError", "EVENT_KINDS",
           "ACQUIRE_KINDS"]
