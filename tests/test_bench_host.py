"""Host logic of bench.py that runs without a GPU: the C3 ``secondary`` leg
(parsed from a fresh process, never fatal for the headline line)."""

import json
import os
import subprocess
import sys
import types

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)

import bench  # noqa: E402


def _args():
    return types.SimpleNamespace(steps=4, warmup=3, weights="reference")


def test_secondary_parses_the_c3_line(monkeypatch):
    c3 = {"value": 29.8, "unit": "tokens/s", "ms_per_step": 33.5, "steps": 4, "warmup": 3,
          "hit_rate": 0.76, "h2d_gbs": 54.1, "miss_loads_per_token": 15.0,
          "spec_loads_per_token": 31.0, "clocks": {"sm_mhz": 1965.0}, "gpu_launches": 640,
          "config": {"workload": "C3: ..."}, "e2e": {"value": 28.5},
          "roofline_e2e": {"frac": 0.92}}
    seen = {}

    def fake_run(cmd, **kw):
        seen["cmd"] = cmd
        return subprocess.CompletedProcess(cmd, 0, "progress\n" + json.dumps(c3) + "\n", "")

    monkeypatch.setattr(bench.subprocess, "run", fake_run)
    out = bench.run_secondary(_args())
    assert "--config" in seen["cmd"] and seen["cmd"][seen["cmd"].index("--config") + 1] == "c3"
    assert "--no-secondary" in seen["cmd"]  # no recursion
    assert out["value"] == 29.8 and out["e2e"]["value"] == 28.5
    assert out["roofline_e2e"]["frac"] == 0.92 and out["config"]["workload"] == "C3: ..."


def test_secondary_failure_is_reported_not_raised(monkeypatch):
    monkeypatch.setattr(bench.subprocess, "run", lambda cmd, **kw: subprocess.CompletedProcess(
        cmd, 3, "", "CUDA error: out of memory"))
    out = bench.run_secondary(_args())
    assert "error" in out and "rc=3" in out["error"]

    def boom(cmd, **kw):
        raise subprocess.TimeoutExpired(cmd, 900)

    monkeypatch.setattr(bench.subprocess, "run", boom)
    assert "TimeoutExpired" in bench.run_secondary(_args())["error"]
