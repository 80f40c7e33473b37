"""The parallel init_params regenerator (paper_2312_17238_b200/initw.py) equals
the reference's serial draw (model.py:145-175, restated by oracle.model), and
the committed Mixtral-shape state table is consistent (CPU)."""

import os
import subprocess
import sys

import numpy as np

from oracle import model as OM
from paper_2312_17238_b200 import initw

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_states_regenerate_init_params(tmp_path):
    cfg = OM.ModelConfig(vocab_size=96, d_model=64, n_layers=3, n_heads=2, d_ffn=128,
                         n_experts=4, max_seq_len=32, seed=5)
    out = tmp_path / "states.json"
    subprocess.run([sys.executable, os.path.join(ROOT, "tools", "make_init_states.py"), str(out),
                    "96", "64", "3", "2", "128", "4", "32", "5"], check=True,
                   capture_output=True)
    doc = initw.load_states(str(out))
    ref = OM.init_params(cfg)
    names = [t["name"] for t in doc["tensors"]]
    assert names[:3] == ["wte", "wpe", "lm_head"] and len(names) == 3 + 3 * (5 + 3 * 4)
    for nm, w in initw.iter_tensors(doc, names, threads=4):
        np.testing.assert_array_equal(w, ref[nm], err_msg=nm)
    assert set(initw.dense_names(3)) | {n for l in range(3) for e in range(4)
                                        for n in initw.expert_names(l, e)} == set(names)


def test_mixtral_state_table():
    doc = initw.load_states()
    c = doc["config"]
    assert (c["vocab_size"], c["d_model"], c["n_layers"], c["n_heads"], c["d_ffn"],
            c["n_experts"], c["max_seq_len"], c["seed"]) == (32000, 4096, 32, 32, 14336, 8, 256, 0)
    assert len(doc["tensors"]) == 3 + 32 * (5 + 3 * 8)
    # the first tensor starts the seed-0 stream; wpe's first draws follow wte's
    rng = np.random.default_rng(0)
    assert int(doc["tensors"][0]["state"]) == rng.bit_generator.state["state"]["state"]
    # wpe's recorded start state is where the serial stream stands after wte
    buf = np.empty(1 << 22)
    n = 32000 * 4096
    while n:
        c = min(n, buf.size)
        rng.standard_normal(out=buf[:c])
        n -= c
    assert int(doc["tensors"][1]["state"]) == rng.bit_generator.state["state"]["state"]
    w = initw.gen_tensor(doc["by_name"]["layers.0.gate"])
    assert w.shape == (4096, 8) and w.dtype == np.float32
    assert abs(float(w.std()) - 1 / 64) < 1e-3
