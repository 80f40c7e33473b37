"""Opt-in B200 backend for the reference package, as a maintainer would wire it
(INTEGRATION.md): importing this module rebinds the reference's session classes
``moe_offload.engine.OffloadEngine`` and ``DenseRunner`` (engine.py:185-247) to
the B200 engine, so every caller of the reference API -- including the
reference's own test suite (``pytest -p paper_2312_17238_b200.refshim``) --
runs on the GPU unchanged.  Loadable as a pytest plugin; it reports how many
B200 engines the session created."""

from __future__ import annotations

from . import api  # noqa: F401  (makes moe_offload importable)
import moe_offload.engine as _ref_engine  # noqa: E402

from . import engine as _b200  # noqa: E402

CREATED = {"OffloadEngine": 0, "DenseRunner": 0}


class OffloadEngine(_b200.OffloadEngine):
    def __init__(self, *a, **kw):
        CREATED["OffloadEngine"] += 1
        super().__init__(*a, **kw)


class DenseRunner(_b200.DenseRunner):
    def __init__(self, *a, **kw):
        CREATED["DenseRunner"] += 1
        super().__init__(*a, **kw)


def install() -> None:
    _ref_engine.OffloadEngine = OffloadEngine
    _ref_engine.DenseRunner = DenseRunner


install()


def pytest_report_header(config):
    return "moe_offload.engine.OffloadEngine / DenseRunner -> paper_2312_17238_b200 (B200 backend)"


def pytest_terminal_summary(terminalreporter, exitstatus, config):
    terminalreporter.write_line(f"B200 backend engines created: OffloadEngine "
                                f"{CREATED['OffloadEngine']}, DenseRunner {CREATED['DenseRunner']}")
