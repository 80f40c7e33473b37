"""Oracle restatement of the reference group quantizer (TEST INFRASTRUCTURE ONLY).

Follows ``/root/reference/pkg/src/moe_offload/quant.py``:
  * schemes / presets ............................. quant.py:34-73
  * LSB-first n-bit packing ....................... quant.py:105-128
  * row padding with the last value ............... quant.py:131-139
  * two-level affine metadata ..................... quant.py:147-178
  * quantize / dequantize ......................... quant.py:181-304
  * bits_per_param / payload_nbytes ............... quant.py:307-343
  * serialized block layout ....................... quant.py:325-421

The arithmetic types are part of the contract and are kept exactly: group
min/max and codes in float32, the zero-point run spread in float64 before the
float16 rounding, one float16 scale per ``scale_group_size`` weights, one
(zscale, zoffset) float16 pair per run of ``scale_group_size`` *groups*.
"""

from __future__ import annotations

import struct
from dataclasses import dataclass

import numpy as np

VALID_BITS = (2, 3, 4, 16)


class QuantFormatError(ValueError):
    """Corrupted or inconsistent block (reference quant.py:30-31)."""


@dataclass(frozen=True)
class QuantScheme:
    """Code width + grouping (reference quant.py:34-63)."""

    bits: int
    group_size: int = 16
    scale_group_size: int = 128
    meta_bits: int = 8
    scale_storage_bits: int = 16

    def __post_init__(self):
        if self.bits not in VALID_BITS:
            raise ValueError(f"bits must be one of {VALID_BITS}")
        if self.bits == 16:
            return
        if self.group_size < 1:
            raise ValueError("group_size must be >= 1")
        if self.scale_group_size % self.group_size:
            raise ValueError("scale_group_size must be a multiple of group_size")
        if not 2 <= self.meta_bits <= 8:
            raise ValueError("meta_bits must be in [2, 8]")
        if self.scale_storage_bits != 16:
            raise ValueError("only 16-bit scale storage is supported")

    @property
    def is_passthrough(self) -> bool:
        return self.bits == 16


SCHEME_FP16 = QuantScheme(16)
SCHEME_4BIT = QuantScheme(4, group_size=64, scale_group_size=256)
SCHEME_3BIT = QuantScheme(3, group_size=64, scale_group_size=128)
SCHEME_2BIT = QuantScheme(2, group_size=16, scale_group_size=128)
PRESETS = {16: SCHEME_FP16, 4: SCHEME_4BIT, 3: SCHEME_3BIT, 2: SCHEME_2BIT}


@dataclass
class QuantizedBlock:
    """Packed codes + metadata (reference quant.py:76-102); field names match
    the reference so either class can be handed to the B200 loader."""

    scheme: QuantScheme
    packed_codes: bytes
    zeros: np.ndarray
    zero_scales: np.ndarray
    zero_offsets: np.ndarray
    scales: np.ndarray
    original_shape: tuple
    pad_count: int = 0

    @property
    def num_weights(self) -> int:
        return int(np.prod(self.original_shape))

    @property
    def padded_count(self) -> int:
        return self.num_weights + self.pad_count


# ---------------------------------------------------------------- bit packing

def pack_bits(codes: np.ndarray, bits: int) -> bytes:
    """Little-endian bitstream, code n occupying bits [n*bits, (n+1)*bits)
    (reference quant.py:105-113).  Eight codes always fill exactly ``bits``
    bytes, so the stream is built eight codes at a time in a uint64."""
    c = np.ascontiguousarray(codes, dtype=np.uint8).reshape(-1)
    if c.size and int(c.max()) >> bits:
        raise ValueError(f"code out of range for {bits}-bit packing")
    if bits == 8:
        return c.tobytes()
    n = c.size
    nbytes = (n * bits + 7) // 8
    c8 = np.concatenate([c, np.zeros((-n) % 8, np.uint8)]).reshape(-1, 8).astype(np.uint64)
    word = np.zeros(c8.shape[0], np.uint64)
    for k in range(8):
        word |= c8[:, k] << np.uint64(bits * k)
    out = word.astype("<u8").view(np.uint8).reshape(-1, 8)[:, :bits]
    return out.reshape(-1)[:nbytes].tobytes()


def unpack_bits(buf: bytes, bits: int, count: int) -> np.ndarray:
    """Inverse of :func:`pack_bits` (reference quant.py:116-128)."""
    raw = np.frombuffer(buf, dtype=np.uint8)
    if bits == 8:
        if raw.size < count:
            raise QuantFormatError("packed buffer shorter than declared code count")
        return raw[:count].copy()
    if raw.size * 8 < count * bits:
        raise QuantFormatError("packed buffer shorter than declared code count")
    ngrp = -(-count // 8)
    need = ngrp * bits
    r = np.zeros(need, np.uint8)
    take = min(need, raw.size)
    r[:take] = raw[:take]
    b = np.zeros((ngrp, 8), np.uint8)
    b[:, :bits] = r.reshape(ngrp, bits)
    word = b.reshape(-1).view("<u8")
    mask = np.uint64((1 << bits) - 1)
    out = np.empty((ngrp, 8), np.uint8)
    for k in range(8):
        out[:, k] = ((word >> np.uint64(bits * k)) & mask).astype(np.uint8)
    return out.reshape(-1)[:count]


# ---------------------------------------------------------------- quantize

def _flatten_padded(w: np.ndarray, g: int):
    """Row-wise padding by repeating the last column (reference quant.py:131-139)."""
    m = w[None, :] if w.ndim == 1 else w
    rows, cols = m.shape
    extra = (-cols) % g
    if extra:
        m = np.concatenate([m, np.repeat(m[:, -1:], extra, axis=1)], axis=1)
    return np.ascontiguousarray(m, dtype=np.float32).reshape(-1), rows * extra


def _quantize_runs(values: np.ndarray, run: int, levels: int):
    """Affine u8 codes for the group minima in runs of ``run`` entries
    (reference quant.py:147-169).  Spread is taken in float64 and the stored
    scale/offset are float16; codes use the exact float32 run minimum."""
    n = values.size
    nruns = -(-n // run)
    pad = nruns * run - n
    v = np.concatenate([values, np.repeat(values[-1:], pad)]) if pad else values
    blocks = v.reshape(nruns, run)
    lo32 = blocks.min(axis=1)                      # float32 minimum per run
    hi32 = blocks.max(axis=1)
    spread = hi32.astype(np.float64) - lo32.astype(np.float64)
    step = np.where(spread > 0.0, spread / (levels - 1), 1.0)
    step16 = step.astype(np.float16)
    c = np.rint((blocks - lo32[:, None]) / step16.astype(np.float32)[:, None])
    codes = np.clip(c, 0, levels - 1).astype(np.uint8).reshape(-1)[:n]
    return codes, step16, lo32.astype(np.float16)


def _dequantize_runs(codes, zscales, zoffsets, run: int) -> np.ndarray:
    """reference quant.py:172-178: code*scale + offset, float32."""
    n = codes.size
    idx = np.arange(n) // run
    return (codes.astype(np.float32) * zscales.astype(np.float32)[idx]
            + zoffsets.astype(np.float32)[idx]).astype(np.float32)


def quantize(w: np.ndarray, scheme: QuantScheme) -> QuantizedBlock:
    """Round-to-nearest affine group quantization (reference quant.py:181-229)."""
    w = np.asarray(w, dtype=np.float32)
    if not np.all(np.isfinite(w)):
        raise ValueError("cannot quantize non-finite values")
    if scheme.is_passthrough:
        raise ValueError("bits=16 is passthrough")
    g, sg = scheme.group_size, scheme.scale_group_size
    top = (1 << scheme.bits) - 1
    flat, pad = _flatten_padded(w, g)
    grp = flat.reshape(-1, g)
    gmin = grp.min(axis=1)
    gmax = grp.max(axis=1)
    gscale = (gmax - gmin) / np.float32(top)       # float32 per-group scale
    per_sg = sg // g
    ngroups = gmin.size
    nsg = -(-ngroups // per_sg)
    padn = nsg * per_sg - ngroups
    gs = np.concatenate([gscale, np.zeros(padn, np.float32)]) if padn else gscale
    smax = gs.reshape(nsg, per_sg).max(axis=1)
    scales = np.where(smax > 0.0, smax, np.float32(1.0)).astype(np.float16)
    s_of_group = np.repeat(scales.astype(np.float32), per_sg)[:ngroups]
    codes = np.rint((grp - gmin[:, None]) / s_of_group[:, None])
    codes = np.clip(codes, 0, top).astype(np.uint8).reshape(-1)
    zc, zs, zo = _quantize_runs(gmin, sg, 1 << scheme.meta_bits)
    return QuantizedBlock(scheme, pack_bits(codes, scheme.bits), zc, zs, zo, scales,
                          tuple(w.shape), pad)


def passthrough(w: np.ndarray) -> QuantizedBlock:
    """16-bit storage (reference quant.py:232-250)."""
    w = np.asarray(w, dtype=np.float32)
    if not np.all(np.isfinite(w)):
        raise ValueError("cannot store non-finite values")
    e8, e16 = np.empty(0, np.uint8), np.empty(0, np.float16)
    return QuantizedBlock(SCHEME_FP16, w.astype(np.float16).tobytes(), e8, e16, e16, e16,
                          tuple(w.shape), 0)


def encode(w: np.ndarray, scheme: QuantScheme) -> QuantizedBlock:
    return passthrough(w) if scheme.is_passthrough else quantize(w, scheme)


def zero_points(block) -> np.ndarray:
    """Reconstructed per-group zeros (reference quant.py:260-264)."""
    return _dequantize_runs(np.asarray(block.zeros), np.asarray(block.zero_scales),
                            np.asarray(block.zero_offsets), block.scheme.scale_group_size)


def dequantize(block) -> np.ndarray:
    """float32 reconstruction: code*scale + zhat (reference quant.py:267-304)."""
    sch = block.scheme
    shape = tuple(block.original_shape)
    n = int(np.prod(shape))
    if sch.bits == 16:
        if len(block.packed_codes) != 2 * n:
            raise QuantFormatError("passthrough payload size mismatch")
        return np.frombuffer(block.packed_codes, np.float16, count=n).astype(np.float32).reshape(shape)
    g, sg = sch.group_size, sch.scale_group_size
    padded = n + block.pad_count
    rows = shape[0] if len(shape) > 1 else 1
    cols = padded // rows
    if padded % g or rows * cols != padded:
        raise QuantFormatError("padded element count inconsistent with group size")
    ngroups = padded // g
    if np.asarray(block.zeros).size != ngroups:
        raise QuantFormatError("zeros length mismatch")
    if np.asarray(block.scales).size != -(-ngroups // (sg // g)):
        raise QuantFormatError("scales length mismatch")
    nz = np.asarray(block.zero_scales).size
    if nz != -(-ngroups // sg) or nz != np.asarray(block.zero_offsets).size:
        raise QuantFormatError("zero metadata length mismatch")
    codes = unpack_bits(block.packed_codes, sch.bits, padded).astype(np.float32)
    zhat = zero_points(block)
    s = np.repeat(np.asarray(block.scales).astype(np.float32), sg // g)[:ngroups]
    vals = (codes.reshape(-1, g) * s[:, None] + zhat[:, None]).reshape(rows, cols)
    keep = cols - (block.pad_count // rows if rows else 0)
    vals = vals[:, :keep]
    return vals.reshape(shape) if len(shape) > 1 else vals.reshape(-1)[:n]


# ---------------------------------------------------------------- accounting

def bits_per_param(scheme: QuantScheme) -> float:
    """reference quant.py:307-318."""
    if scheme.is_passthrough:
        return 16.0
    g, sg, s = scheme.group_size, scheme.scale_group_size, scheme.scale_storage_bits
    return scheme.bits + scheme.meta_bits / g + s / sg + 2 * s / (g * sg)


def payload_nbytes(block) -> int:
    """Serialized payload bytes excluding the header (reference quant.py:332-343)
    — this is the H2D byte count of one matrix."""
    if block.scheme.is_passthrough:
        return len(block.packed_codes)
    zb = -(-np.asarray(block.zeros).size * block.scheme.meta_bits // 8)
    return (len(block.packed_codes) + zb + 2 * np.asarray(block.zero_scales).size
            + 2 * np.asarray(block.zero_offsets).size + 2 * np.asarray(block.scales).size)


_HDR = "<BBIIBB"


def serialize(block) -> bytes:
    """Header, codes, zeros, zscales, zoffsets, scales (reference quant.py:346-365)."""
    s = block.scheme
    pt = s.is_passthrough
    parts = [struct.pack(_HDR, 1, s.bits, 0 if pt else s.group_size,
                         0 if pt else s.scale_group_size, 0 if pt else s.meta_bits,
                         len(block.original_shape))]
    parts += [struct.pack("<I", d) for d in block.original_shape]
    parts.append(struct.pack("<I", block.pad_count))
    parts.append(bytes(block.packed_codes))
    if not pt:
        parts.append(pack_bits(np.asarray(block.zeros), s.meta_bits))
        for arr in (block.zero_scales, block.zero_offsets, block.scales):
            parts.append(np.asarray(arr).astype("<f2").tobytes())
    return b"".join(parts)


def deserialize(buf: bytes) -> QuantizedBlock:
    """reference quant.py:368-421."""
    base = struct.calcsize(_HDR)
    if len(buf) < base:
        raise QuantFormatError("buffer shorter than header")
    ver, bits, g, sg, mb, ndim = struct.unpack_from(_HDR, buf, 0)
    if ver != 1:
        raise QuantFormatError("unsupported version")
    if bits not in VALID_BITS:
        raise QuantFormatError("unsupported code width")
    off = base
    if len(buf) < off + 4 * ndim + 4:
        raise QuantFormatError("buffer shorter than declared shape")
    shape = tuple(struct.unpack_from(f"<{ndim}I", buf, off)) if ndim else ()
    off += 4 * ndim
    (pad,) = struct.unpack_from("<I", buf, off)
    off += 4
    n = int(np.prod(shape)) if shape else 0
    if bits == 16:
        body = buf[off:off + 2 * n]
        if len(body) != 2 * n:
            raise QuantFormatError("truncated passthrough payload")
        e8, e16 = np.empty(0, np.uint8), np.empty(0, np.float16)
        return QuantizedBlock(SCHEME_FP16, body, e8, e16, e16, e16, shape, 0)
    sch = QuantScheme(bits, group_size=g, scale_group_size=sg, meta_bits=mb)
    padded = n + pad
    if g == 0 or padded % g:
        raise QuantFormatError("pad_count inconsistent with group size")
    ng = padded // g
    nsg = -(-ng // (sg // g))
    nz = -(-ng // sg)
    cb = -(-padded * bits // 8)
    zb = -(-ng * mb // 8)
    if len(buf) - off != cb + zb + 4 * nz + 2 * nsg:
        raise QuantFormatError("payload length does not match layout")
    codes = buf[off:off + cb]
    off += cb
    zeros = unpack_bits(buf[off:off + zb], mb, ng)
    off += zb
    zs = np.frombuffer(buf, "<f2", nz, off).copy()
    off += 2 * nz
    zo = np.frombuffer(buf, "<f2", nz, off).copy()
    off += 2 * nz
    sc = np.frombuffer(buf, "<f2", nsg, off).copy()
    return QuantizedBlock(sch, codes, zeros, zs, zo, sc, shape, pad)
