"""Serialized quant blocks (quant.serialize_block bytes) parsed by the C ABI
(csrc/blockio.cu, moe_parse_block) exactly like the reference's
deserialize_block (quant.py:364-421): same fields on the golden blocks the
unmodified reference serialized (tests/golden/quant_golden.npz) and on fresh
ones, the same QuantFormatError messages on malformed input.  CPU only."""

import ctypes as C
import struct

import numpy as np
import pytest

from paper_2312_17238_b200 import _lib
from paper_2312_17238_b200.api import moe_offload  # noqa: F401
from moe_offload import quant as RQ


def _parse(buf: bytes):
    L = _lib.lib()
    m = _lib.Matrix()
    ng = C.c_int64()
    _lib.check(L.moe_parse_block(buf, len(buf), C.byref(m), None, 0, C.byref(ng)))
    z = np.zeros(max(ng.value, 1), np.uint8)
    _lib.check(L.moe_parse_block(buf, len(buf), C.byref(m), z.ctypes.data_as(C.c_void_p),
                                 ng.value, C.byref(ng)))
    return m, z[:ng.value]


def _f16(ptr, n):
    return np.ctypeslib.as_array(C.cast(ptr, C.POINTER(C.c_uint16)), (n,)).copy() if n else \
        np.zeros(0, np.uint16)


def _check_same(buf: bytes):
    ref = RQ.deserialize_block(buf)
    m, z = _parse(buf)
    assert (m.rows, m.cols) == tuple(ref.original_shape)
    assert m.bits == ref.scheme.bits
    codes = C.string_at(m.codes, m.codes_len)
    assert codes == bytes(ref.packed_codes)
    if ref.scheme.bits == 16:
        return
    assert (m.group_size, m.scale_group_size, m.meta_bits, m.pad_count) == (
        ref.scheme.group_size, ref.scheme.scale_group_size, ref.scheme.meta_bits, ref.pad_count)
    np.testing.assert_array_equal(z, ref.zeros)
    np.testing.assert_array_equal(_f16(m.zero_scales, m.n_zruns), ref.zero_scales.view(np.uint16))
    np.testing.assert_array_equal(_f16(m.zero_offsets, m.n_zruns),
                                  ref.zero_offsets.view(np.uint16))
    np.testing.assert_array_equal(_f16(m.scales, m.n_scales), ref.scales.view(np.uint16))


def test_golden_blocks_parse_like_reference():
    g = np.load("tests/golden/quant_golden.npz")
    n = 0
    for key in g.files:
        if key.startswith("ser"):
            _check_same(g[key].tobytes())
            n += 1
    assert n >= 8


@pytest.mark.parametrize("bits", [2, 3, 4, 16])
@pytest.mark.parametrize("shape", [(64, 256), (48, 40), (7, 9)])
def test_fresh_blocks_parse_like_reference(bits, shape):
    w = np.random.default_rng(bits * 100 + shape[0]).normal(0, 0.05, shape).astype(np.float32)
    blk = RQ.passthrough_block(w) if bits == 16 else RQ.quantize(w, RQ.PRESET_SCHEMES[bits])
    _check_same(RQ.serialize_block(blk))


def _ref_error(buf):
    with pytest.raises(RQ.QuantFormatError) as e:
        RQ.deserialize_block(buf)
    return str(e.value)


def test_malformed_blocks_raise_reference_errors():
    w = np.random.default_rng(0).normal(0, 0.05, (32, 64)).astype(np.float32)
    good = RQ.serialize_block(RQ.quantize(w, RQ.PRESET_SCHEMES[3]))
    bad = [good[:5],                                   # shorter than the header
           bytes([9]) + good[1:],                      # version
           good[:1] + bytes([5]) + good[2:],           # code width
           good[:14],                                  # shape truncated
           good[:-3],                                  # payload length
           good + b"\0\0"]
    for b in bad:
        msg = _ref_error(b)
        with pytest.raises(RQ.QuantFormatError) as e:
            _parse(b)
        assert str(e.value) == msg
    # pad_count inconsistent with the group size
    hdr = struct.calcsize("<BBIIBB") + 8
    b = bytearray(good)
    struct.pack_into("<I", b, hdr, 3)
    msg = _ref_error(bytes(b))
    with pytest.raises(RQ.QuantFormatError) as e:
        _parse(bytes(b))
    assert str(e.value) == msg
