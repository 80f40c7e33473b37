"""Pins the oracle's quantizer to the reference (CPU; no GPU needed).

Golden vectors (tests/golden/quant_golden.npz) were produced by the unmodified
reference ``moe_offload.quant`` (tests/golden/make_golden.py); the known-answer
tests restate the reference's own (pkg/tests/test_quant.py:113-192).
"""

import hashlib
import os

import numpy as np
import pytest

from oracle import quant as OQ

GOLDEN = os.path.join(os.path.dirname(__file__), "golden")
CASES = [  # must match make_golden.QUANT_CASES
    (2, (128, 128), 42, 1.0), (3, (64, 256), 1, 0.3), (4, (64, 1024), 2, 0.05),
    (2, (7, 33), 3, 2.0), (3, (5, 200), 4, 1.0), (4, (16, 100), 5, 10.0),
    (2, (256, 896), 6, 1 / 16), (3, (256, 896), 7, 1 / 16), (4, (256, 256), 8, 1 / 16),
    (2, (896, 256), 9, 1 / 30), (3, (896, 256), 10, 1 / 30),
]


@pytest.fixture(scope="module")
def golden():
    return np.load(os.path.join(GOLDEN, "quant_golden.npz"))


@pytest.mark.parametrize("i", range(len(CASES)))
def test_quantize_bytes_match_reference(i, golden):
    bits, shape, seed, scale = CASES[i]
    assert int(golden["bits"][i]) == bits
    w = (np.random.default_rng(seed).normal(size=shape) * scale).astype(np.float32)
    blk = OQ.quantize(w, OQ.PRESETS[bits])
    assert OQ.serialize(blk) == golden[f"ser{i}"].tobytes()
    assert OQ.payload_nbytes(blk) == int(golden[f"nbytes{i}"])
    deq = OQ.dequantize(blk).astype("<f4").tobytes()
    assert hashlib.sha256(deq).digest() == golden[f"deq_sha{i}"].tobytes()


@pytest.mark.parametrize("i", range(len(CASES)))
def test_deserialize_reference_bytes(i, golden):
    buf = golden[f"ser{i}"].tobytes()
    blk = OQ.deserialize(buf)
    assert OQ.serialize(blk) == buf
    deq = OQ.dequantize(blk).astype("<f4").tobytes()
    assert hashlib.sha256(deq).digest() == golden[f"deq_sha{i}"].tobytes()


def test_2bit_regression_checksum():
    """reference test_quant.py:113-120."""
    w = np.random.default_rng(42).normal(size=(128, 128)).astype(np.float32)
    blk = OQ.quantize(w, OQ.SCHEME_2BIT)
    err = float(np.abs(OQ.dequantize(blk) - w).mean())
    assert err == pytest.approx(0.36625814, abs=1e-6)


def test_bits_per_param_and_byte_counts():
    """reference test_quant.py:183-200 and SURVEY §8 expert byte counts."""
    assert OQ.bits_per_param(OQ.SCHEME_2BIT) == 2.640625
    assert OQ.bits_per_param(OQ.SCHEME_3BIT) == 3.25390625
    assert OQ.bits_per_param(OQ.SCHEME_4BIT) == 4.189453125
    w = np.zeros((256, 512), np.float32)
    for sch in (OQ.SCHEME_2BIT, OQ.SCHEME_3BIT, OQ.SCHEME_4BIT):
        blk = OQ.quantize(w, sch)
        assert OQ.payload_nbytes(blk) * 8 == OQ.bits_per_param(sch) * w.size


def test_mixtral_expert_bytes():
    """payload_nbytes of one Mixtral-shape expert without materialising it."""
    import bench
    assert bench.expert_bytes(bench.MIXTRAL, 2) == 58_146_816
    assert bench.expert_bytes(bench.MIXTRAL, 3) == 71_651_328
    assert bench.expert_bytes(bench.MIXTRAL, 4) == 92_252_160
    assert 4 * bench.matrix_payload_bytes(4096, 4096, 4) == 35_143_680


def test_3bit_exhaustive_8code_windows():
    """Every 8-code window packs to the 3-byte little-endian integer
    (reference test_quant.py:158-172)."""
    v = np.arange(1 << 24, dtype=np.uint32)
    codes = np.stack([(v >> (3 * k)) & 7 for k in range(8)], axis=1).astype(np.uint8)
    buf = OQ.pack_bits(codes.reshape(-1), 3)
    raw = np.frombuffer(buf, np.uint8).reshape(-1, 3).astype(np.uint32)
    assert np.array_equal(raw[:, 0] | (raw[:, 1] << 8) | (raw[:, 2] << 16), v)
    back = OQ.unpack_bits(buf, 3, codes.size)
    assert np.array_equal(back, codes.reshape(-1))


@pytest.mark.parametrize("bits", [2, 3, 4, 8])
def test_pack_unpack_bijective(bits):
    rng = np.random.default_rng(bits)
    for n in (1, 7, 8, 9, 100, 1001):
        c = rng.integers(0, 1 << bits, n).astype(np.uint8)
        assert np.array_equal(OQ.unpack_bits(OQ.pack_bits(c, bits), bits, n), c)


def test_rejects_out_of_range_and_nonfinite():
    with pytest.raises(ValueError):
        OQ.pack_bits(np.array([4], np.uint8), 2)
    with pytest.raises(ValueError):
        OQ.quantize(np.array([[np.nan, 1.0]], np.float32), OQ.SCHEME_2BIT)
    with pytest.raises(ValueError):
        OQ.quantize(np.ones((2, 2), np.float32), OQ.SCHEME_FP16)


def test_idempotent_on_lattice():
    """reference test_quant.py:87-93."""
    w = np.random.default_rng(3).normal(size=(64, 256)).astype(np.float32)
    for sch in (OQ.SCHEME_2BIT, OQ.SCHEME_3BIT, OQ.SCHEME_4BIT):
        b1 = OQ.quantize(w, sch)
        b2 = OQ.quantize(OQ.dequantize(b1), sch)
        assert OQ.serialize(b1) == OQ.serialize(b2)


def test_constant_matrix_exact():
    w = np.full((8, 128), 0.75, np.float32)
    for sch in (OQ.SCHEME_2BIT, OQ.SCHEME_3BIT, OQ.SCHEME_4BIT):
        assert np.array_equal(OQ.dequantize(OQ.quantize(w, sch)), w)


def test_corrupted_payload_rejected():
    w = np.random.default_rng(0).normal(size=(16, 64)).astype(np.float32)
    buf = OQ.serialize(OQ.quantize(w, OQ.SCHEME_2BIT))
    with pytest.raises(OQ.QuantFormatError):
        OQ.deserialize(buf[:-1])
    with pytest.raises(OQ.QuantFormatError):
        OQ.deserialize(b"\x02" + buf[1:])


def test_dequant_exact_in_fp32_regardless_of_fma():
    """code*scale + zhat is exact in fp32 for every preset (the property that
    lets the device GEMV reproduce dequantized weights bit for bit)."""
    rng = np.random.default_rng(9)
    for sch in (OQ.SCHEME_2BIT, OQ.SCHEME_3BIT, OQ.SCHEME_4BIT):
        w = (rng.normal(size=(32, 512)) / 20).astype(np.float32)
        blk = OQ.quantize(w, sch)
        codes = OQ.unpack_bits(blk.packed_codes, sch.bits, w.size).astype(np.float64)
        s = np.repeat(blk.scales.astype(np.float64), sch.scale_group_size // sch.group_size)
        z = OQ.zero_points(blk).astype(np.float64)
        exact = (codes.reshape(-1, sch.group_size) * s[:, None] + z[:, None]).reshape(w.shape)
        assert np.array_equal(exact.astype(np.float32).astype(np.float64), exact)
        assert np.array_equal(OQ.dequantize(blk), exact.astype(np.float32))
