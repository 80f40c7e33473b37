"""The C-ABI library loads and exports exactly what include/moeb200.h declares
(CPU: no compute calls), and the Python mirror keeps the reference API."""

import ctypes as C
import os
import re

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "moeb200.h")


def header_functions():
    src = open(HEADER).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return set(re.findall(r"^\s*(?:const\s+)?[a-z_0-9]+\s*\*?\s*(moe_[a-z_0-9]+)\s*\(", src,
                          flags=re.M))


@pytest.fixture(scope="module")
def lib():
    from paper_2312_17238_b200 import _lib
    if not os.path.exists(_lib.LIB_PATH):
        from paper_2312_17238_b200 import build
        build.build()
    return _lib.lib()


def test_header_and_binding_agree():
    from paper_2312_17238_b200 import _lib
    fns = header_functions()
    assert len(fns) >= 20
    assert fns == set(_lib.SIGNATURES), fns ^ set(_lib.SIGNATURES)


def test_library_exports_every_symbol(lib):
    for name in header_functions():
        assert hasattr(lib, name), name


def test_struct_layouts_match_header():
    from paper_2312_17238_b200 import _lib
    assert C.sizeof(_lib.Event) == 32
    assert C.sizeof(_lib.TraceRec) == 72
    assert C.sizeof(_lib.Matrix) == 4 * 7 + 4 + 8 * 9
    assert C.sizeof(_lib.ModelDesc) == 32


def test_errors_map_without_gpu(lib):
    """No device here: engine creation fails loudly (no CPU fallback)."""
    import torch
    if torch.cuda.is_available():
        pytest.skip("CPU-only check")
    from paper_2312_17238_b200 import CacheConfig, OffloadEngine, SpeculationConfig
    from oracle import model as OM
    cfg = OM.ModelConfig(vocab_size=32, d_model=32, n_layers=1, n_heads=2, d_ffn=48, n_experts=4)
    with pytest.raises(RuntimeError):
        OffloadEngine(OM.Model(cfg, OM.init_params(cfg)), CacheConfig(2, 4),
                      SpeculationConfig())
    assert isinstance(lib.moe_last_error(), bytes)


def test_status_mapping(lib):
    from paper_2312_17238_b200 import NonFiniteError, QuantFormatError, UnknownExpertError, _lib
    _lib.check(0)
    for rc, exc in [(1, ValueError), (2, RuntimeError), (3, NonFiniteError),
                    (4, UnknownExpertError), (5, QuantFormatError), (6, RuntimeError),
                    (7, RuntimeError)]:
        with pytest.raises(exc):
            _lib.check(rc)


def test_reference_value_types():
    from paper_2312_17238_b200 import (CacheConfig, ExpertKey, SpeculationConfig, StoreEvent,
                                       events_from_jsonl, events_to_jsonl, recall)
    with pytest.raises(ValueError):
        CacheConfig(k=-1)
    with pytest.raises(ValueError):
        SpeculationConfig(lookahead=0)
    ev = [StoreEvent(0, "miss_load", ExpertKey(0, 1), 0, 64),
          StoreEvent(1, "hit", ExpertKey(0, 1), 1, 0),
          StoreEvent(2, "staging_hit", ExpertKey(1, 2), 1, 0),
          StoreEvent(3, "speculative_load", ExpertKey(1, 3), 1, 64)]
    assert events_from_jsonl(events_to_jsonl(ev)) == ev
    assert recall(ev) == pytest.approx(2 / 3)
    assert recall(ev, "device_only") == pytest.approx(1 / 3)
    with pytest.raises(ValueError):
        recall(ev[3:])
    line = events_to_jsonl(ev[:1]).strip()
    assert line == ('{"bytes_moved":64,"expert":1,"kind":"miss_load","layer":0,"seq":0,'
                    '"token_pos":0}')


def test_reference_jsonl_compatible():
    """Our events JSONL equals the reference encoder's (store.py:243-251)."""
    import sys
    ref = "/root/reference/pkg/src"
    if not os.path.isdir(ref):
        pytest.skip("reference not mounted")
    sys.path.insert(0, ref)
    try:
        from moe_offload import store as RS
    finally:
        sys.path.remove(ref)
    from paper_2312_17238_b200 import ExpertKey, StoreEvent, events_to_jsonl
    ev = [StoreEvent(i, k, ExpertKey(i % 2, i % 8), i, 64 * (i % 2)) for i, k in
          enumerate(["hit", "miss_load", "evict_to_host", "promote_from_staging"])]
    rev = [RS.StoreEvent(e.seq, e.kind, RS.ExpertKey(*e.key), e.token_pos, e.bytes_moved)
           for e in ev]
    assert events_to_jsonl(ev) == RS.events_to_jsonl(rev)


def test_payload_nbytes_of_blocks():
    from oracle import quant as OQ
    from paper_2312_17238_b200 import payload_nbytes
    w = np.random.default_rng(0).normal(size=(64, 128)).astype(np.float32)
    trip = tuple(OQ.quantize(w, OQ.SCHEME_2BIT) for _ in range(3))
    assert payload_nbytes(trip) == 3 * OQ.payload_nbytes(trip[0])
