"""Pins the C oracle (oracle/c/oracle.c via oracle/fastq.py) to the reference
golden vectors and to the numpy restatement (CPU; no GPU needed).

quantize must be byte-identical to reference quant.quantize, dequantize
bit-identical to quant.dequantize, gemv equal to x @ dequantize(W) to float64
rounding.
"""

import hashlib
import os

import numpy as np
import pytest

from oracle import fastq as FQ
from oracle import quant as OQ
from tests.test_oracle_quant import CASES

GOLDEN = os.path.join(os.path.dirname(__file__), "golden")


@pytest.fixture(scope="module")
def golden():
    return np.load(os.path.join(GOLDEN, "quant_golden.npz"))


def test_half_conversions_match_numpy():
    rng = np.random.default_rng(0)
    f = np.concatenate([rng.normal(size=20000).astype(np.float32) * 10.0 ** rng.integers(-9, 6, 20000),
                        np.array([0.0, -0.0, 65504, 65520, 65519.99, 1e-8, 2 ** -24, 2 ** -25,
                                  3 * 2 ** -26, 1 + 2 ** -11, 1 + 3 * 2 ** -11], np.float32)])
    f = f.astype(np.float32)
    got = np.array([FQ.lib().oq_f2h(float(v)) for v in f], np.uint16)
    np.testing.assert_array_equal(got, f.astype(np.float16).view(np.uint16))
    d = rng.normal(size=20000) * 10.0 ** rng.integers(-9, 5, 20000)
    d = np.concatenate([d, [1 + 2 ** -11, 1 + 2 ** -11 + 2 ** -40, 2 ** -24 * 1.5, 65519.999]])
    got = np.array([FQ.lib().oq_d2h(float(v)) for v in d], np.uint16)
    np.testing.assert_array_equal(got, d.astype(np.float16).view(np.uint16))


@pytest.mark.parametrize("i", [i for i, c in enumerate(CASES) if c[1][1] % OQ.PRESETS[c[0]].group_size == 0])
def test_c_quantize_matches_reference_golden(i, golden):
    bits, shape, seed, scale = CASES[i]
    w = (np.random.default_rng(seed).normal(size=shape) * scale).astype(np.float32)
    blk = FQ.quantize(w, OQ.PRESETS[bits], nthreads=3)
    assert OQ.serialize(blk) == golden[f"ser{i}"].tobytes()
    deq = FQ.dequantize(blk, nthreads=2).astype("<f4").tobytes()
    assert hashlib.sha256(deq).digest() == golden[f"deq_sha{i}"].tobytes()


@pytest.mark.parametrize("bits,shape,scale", [
    (2, (64, 512), 1.0), (3, (32, 14336), 1 / 64), (4, (96, 4096), 0.02), (3, (448, 128), 3.0),
    (2, (16, 4096), 1e-3), (4, (8, 64), 100.0)])
def test_c_quantize_matches_numpy_oracle(bits, shape, scale):
    rng = np.random.default_rng(bits * 1000 + shape[0])
    w = (rng.normal(size=shape) * scale).astype(np.float32)
    w[0, :] = w[0, 0]  # a constant row: zero spread groups (scale 1.0 path)
    sch = OQ.PRESETS[bits]
    ref = OQ.quantize(w, sch)
    got = FQ.quantize(w, sch, nthreads=4)
    assert got.packed_codes == ref.packed_codes
    np.testing.assert_array_equal(got.zeros, ref.zeros)
    np.testing.assert_array_equal(got.zero_scales.view(np.uint16), ref.zero_scales.view(np.uint16))
    np.testing.assert_array_equal(got.zero_offsets.view(np.uint16),
                                  ref.zero_offsets.view(np.uint16))
    np.testing.assert_array_equal(got.scales.view(np.uint16), ref.scales.view(np.uint16))
    np.testing.assert_array_equal(FQ.dequantize(ref).view(np.uint32),
                                  OQ.dequantize(ref).view(np.uint32))


@pytest.mark.parametrize("bits", [2, 3, 4, 32])
def test_c_gemv_matches_float64_matmul(bits):
    rng = np.random.default_rng(bits)
    K, N = 384, 640
    w = (rng.normal(size=(K, N)) / 20).astype(np.float32)
    X = rng.normal(size=(5, K)).astype(np.float32)
    if bits == 32:
        blk, deq = FQ.dense_block(w), w
    else:
        blk = OQ.quantize(w, OQ.PRESETS[bits])
        deq = OQ.dequantize(blk)
    Y = FQ.gemv(blk, X, nthreads=3)
    ref = X.astype(np.float64) @ deq.astype(np.float64)
    np.testing.assert_allclose(Y, ref, rtol=1e-12, atol=1e-12)
    np.testing.assert_allclose(FQ.gemv(blk, X[2]), ref[2], rtol=1e-12, atol=1e-12)
