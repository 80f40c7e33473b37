"""Opt-in B200 backend for the reference package, as a maintainer would wire it
(INTEGRATION.md): importing this module rebinds the reference's session classes
``moe_offload.engine.OffloadEngine`` and ``DenseRunner`` (engine.py:185-247) to
the B200 engine, so every caller of the reference API -- including the
reference's own test suite (``pytest -p paper_2312_17238_b200.refshim``) --
runs on the GPU unchanged.  Loadable as a pytest plugin."""

from __future__ import annotations

from . import api  # noqa: F401  (makes moe_offload importable)
import moe_offload.engine as _ref_engine  # noqa: E402

from .engine import DenseRunner, OffloadEngine  # noqa: E402


def install() -> None:
    _ref_engine.OffloadEngine = OffloadEngine
    _ref_engine.DenseRunner = DenseRunner


install()


def pytest_report_header(config):
    return (f"moe_offload.engine.OffloadEngine -> {_ref_engine.OffloadEngine.__module__}."
            f"{_ref_engine.OffloadEngine.__name__} (B200 backend)")
