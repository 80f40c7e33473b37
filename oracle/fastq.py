"""ctypes front of the C oracle ``oracle/c/oracle.c`` (TEST INFRASTRUCTURE ONLY).

Same results as the numpy restatement in ``oracle/quant.py`` -- byte-identical
``quantize`` (reference quant.py:181-229), bit-identical ``dequantize``
(quant.py:267-304) -- at C speed and multi-threaded, so that Mixtral-shape
checks and the CPU reference arm finish in seconds per matrix instead of
minutes.  ``gemv`` is x @ dequantize(W) (model.py:223-226, 290-300) fused and
accumulated in float64.  Pinned by tests/test_oracle_c.py.
"""

from __future__ import annotations

import ctypes as C
import os
import subprocess

import numpy as np

from . import quant as Q

HERE = os.path.dirname(os.path.abspath(__file__))
LIB = os.path.join(HERE, "liboracle.so")
_lib = None


class Block(C.Structure):
    _fields_ = [("codes", C.c_void_p), ("zeros", C.c_void_p), ("zs", C.c_void_p),
                ("zo", C.c_void_p), ("scales", C.c_void_p), ("K", C.c_int64),
                ("N", C.c_int64), ("bits", C.c_int), ("g", C.c_int), ("sg", C.c_int)]


def build() -> str:
    src = os.path.join(HERE, "c", "oracle.c")
    if not os.path.exists(LIB) or os.path.getmtime(LIB) < os.path.getmtime(src):
        subprocess.run(["make", "-s", "-C", HERE], check=True)
    return LIB


def lib():
    global _lib
    if _lib is None:
        build()
        L = C.CDLL(LIB)
        vp, i64 = C.c_void_p, C.c_int64
        L.oq_quantize.argtypes = [vp, i64, i64, C.c_int, C.c_int, C.c_int, vp, vp, vp, vp, vp,
                                  C.c_int]
        L.oq_dequantize.argtypes = [C.POINTER(Block), vp, C.c_int]
        L.oq_gemv.argtypes = [C.POINTER(Block), vp, C.c_int, vp, C.c_int]
        L.oq_f2h.argtypes = [C.c_float]
        L.oq_f2h.restype = C.c_uint16
        L.oq_d2h.argtypes = [C.c_double]
        L.oq_d2h.restype = C.c_uint16
        _lib = L
    return _lib


def threads() -> int:
    return int(os.environ.get("ORACLE_THREADS", os.cpu_count() or 1))


def _p(a):
    return a.ctypes.data_as(C.c_void_p)


def quantize_arrays(w: np.ndarray, scheme, nthreads: int | None = None):
    """(codes u8, zeros u8, zero_scales f16, zero_offsets f16, scales f16)."""
    w = np.ascontiguousarray(w, dtype=np.float32)
    if not np.all(np.isfinite(w)):
        raise ValueError("cannot quantize non-finite values")
    K, N = (w.shape if w.ndim == 2 else (1, w.size))
    bits, g, sg = scheme.bits, scheme.group_size, scheme.scale_group_size
    if N % g:
        raise ValueError("C oracle quantizer needs cols % group_size == 0 (no row padding)")
    n = K * N
    ng = n // g
    codes = np.empty((n * bits + 7) // 8, np.uint8)
    zeros = np.empty(ng, np.uint8)
    nr = -(-ng // sg)
    nsg = -(-ng // (sg // g))
    zs, zo, sc = np.empty(nr, np.uint16), np.empty(nr, np.uint16), np.empty(nsg, np.uint16)
    rc = lib().oq_quantize(_p(w), K, N, bits, g, sg, _p(codes), _p(zeros), _p(zs), _p(zo),
                           _p(sc), nthreads or threads())
    if rc:
        raise RuntimeError(f"oq_quantize failed ({rc})")
    return codes, zeros, zs.view(np.float16), zo.view(np.float16), sc.view(np.float16)


def quantize(w: np.ndarray, scheme, nthreads: int | None = None) -> Q.QuantizedBlock:
    """Byte-identical to quant.quantize (no row padding)."""
    codes, zeros, zs, zo, sc = quantize_arrays(w, scheme, nthreads)
    return Q.QuantizedBlock(scheme, codes.tobytes(), zeros, zs, zo, sc, tuple(w.shape), 0)


class _Keep:
    """A Block struct plus the arrays it points into."""

    def __init__(self, block):
        sch = block.scheme
        shape = tuple(block.original_shape)
        K, N = (shape if len(shape) == 2 else (1, int(np.prod(shape))))
        if block.pad_count:
            raise ValueError("C oracle handles unpadded blocks only")
        self.codes = np.frombuffer(block.packed_codes, np.uint8)
        b = Block()
        b.codes = self.codes.ctypes.data
        b.K, b.N, b.bits = K, N, sch.bits
        if sch.bits <= 4:
            self.z = np.ascontiguousarray(block.zeros, np.uint8)
            self.zs = np.ascontiguousarray(block.zero_scales, np.float16)
            self.zo = np.ascontiguousarray(block.zero_offsets, np.float16)
            self.sc = np.ascontiguousarray(block.scales, np.float16)
            b.zeros, b.zs, b.zo, b.scales = (a.ctypes.data for a in (self.z, self.zs, self.zo,
                                                                     self.sc))
            b.g, b.sg = sch.group_size, sch.scale_group_size
        self.b = b
        self.shape = shape


def dense_block(w: np.ndarray):
    """A float32 matrix in the Block form (bits 32) for gemv."""
    w = np.ascontiguousarray(w, np.float32)
    k = _Keep.__new__(_Keep)
    k.codes = w
    b = Block()
    b.codes = w.ctypes.data
    b.K, b.N = w.shape
    b.bits = 32
    k.b, k.shape = b, w.shape
    return k


def dequantize(block, nthreads: int | None = None) -> np.ndarray:
    """Bit-identical to quant.dequantize for 2/3/4-bit blocks."""
    if block.scheme.bits == 16:
        return Q.dequantize(block)
    k = _Keep(block)
    out = np.empty(int(k.b.K * k.b.N), np.float32)
    lib().oq_dequantize(C.byref(k.b), _p(out), nthreads or threads())
    return out.reshape(k.shape)


def gemv(block_or_keep, X: np.ndarray, nthreads: int | None = None) -> np.ndarray:
    """X (n, K) or (K,) @ dequantize(W) in float64 accumulation -> float64."""
    k = block_or_keep if isinstance(block_or_keep, _Keep) else _Keep(block_or_keep)
    X = np.ascontiguousarray(X, np.float32)
    one = X.ndim == 1
    X2 = X[None, :] if one else X
    if X2.shape[1] != k.b.K:
        raise ValueError("shape mismatch")
    Y = np.empty((X2.shape[0], int(k.b.N)), np.float64)
    for s in range(0, X2.shape[0], 64):
        xs = np.ascontiguousarray(X2[s:s + 64])
        ys = np.empty((xs.shape[0], int(k.b.N)), np.float64)
        rc = lib().oq_gemv(C.byref(k.b), _p(xs), xs.shape[0], _p(ys), nthreads or threads())
        if rc:
            raise RuntimeError("oq_gemv failed")
        Y[s:s + 64] = ys
    return Y[0] if one else Y


def prepared(block):
    """Keep-alive Block view for repeated gemv calls on one matrix."""
    return _Keep(block)
