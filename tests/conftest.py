import json
import os
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)
GOLDEN = os.path.join(ROOT, "tests", "golden")


def pytest_sessionstart(session):
    """Install the unmodified reference into baseline/_ref when it is missing
    (the package imports its value types from moe_offload), then (re)build
    libmoeb200.so when a source is newer (no-op otherwise)."""
    if (not os.path.isdir(os.path.join(ROOT, "baseline", "_ref", "moe_offload"))
            and os.path.isdir("/root/reference/pkg")):
        import subprocess
        subprocess.run(["bash", os.path.join(ROOT, "tools", "install_reference.sh")], check=True)
    from paper_2312_17238_b200 import build
    build.build()


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200) and libmoeb200.so")


def pytest_collection_modifyitems(config, items):
    try:
        import torch
        has_gpu = torch.cuda.is_available()
    except Exception:  # pragma: no cover
        has_gpu = False
    if has_gpu:
        return
    skip = pytest.mark.skip(reason="no CUDA device")
    for it in items:
        if "gpu" in it.keywords:
            it.add_marker(skip)


@pytest.fixture(scope="session")
def engine_golden():
    data = np.load(os.path.join(GOLDEN, "engine_golden.npz"))
    with open(os.path.join(GOLDEN, "engine_cases.json")) as fh:
        meta = json.load(fh)
    return data, meta


@pytest.fixture(scope="session")
def c1_models():
    """C1-family models from the oracle (init_params + mixed quant), cached."""
    from oracle import engine as OE
    from oracle import model as OM
    with open(os.path.join(GOLDEN, "engine_cases.json")) as fh:
        cfg = OM.ModelConfig(**json.load(fh)["config"])
    params = OM.init_params(cfg)
    cache = {}

    def get(q):
        if q not in cache:
            if q is None:
                cache[q] = (OM.Model(cfg, params), None, None)
            else:
                fq, pay, attn = OE.build_mixed_quant(params, cfg, *q)
                cache[q] = (OM.Model(cfg, fq), pay, attn)
        return cache[q]
    return cfg, get


def make_prompt(seed, length, vocab):
    rng = np.random.default_rng(seed)
    return [int(t) for t in rng.integers(0, vocab, size=length)]
