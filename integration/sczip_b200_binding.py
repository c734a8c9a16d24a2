"""The binding a `sczip` maintainer adds to route the hot path to the GPU.

Install as ``sczip/_b200.py`` in the reference package (next to
container.py) and add the three-line hook shown in INTEGRATION.md to
``container.compress`` / ``container.decompress``.  It binds the C ABI of
include/sczip_b200.h with ctypes only -- no torch, no paper_2511_11664_b200
import -- and returns the reference's own ``Container`` / ``FeatureTensor``
objects.  tests/test_integration_binding.py executes this file against the
drop-in package standing in for ``sczip``.

Entry points bound (header line -> reference function replaced):
  scz_ctx_create / scz_last_error            (context, error text)
  scz_compress    -> container.compress      container.py:73-106
  scz_decompress  -> container.decompress    container.py:109-121
"""

from __future__ import annotations

import ctypes
import os

import numpy as np

from . import errors, optimizer
from .container import Container
from .tensor import FeatureTensor, QuantParams

_LIB_NAME = os.environ.get("SCZIP_B200_LIB", "libsczip_b200.so")
_lib = ctypes.CDLL(_LIB_NAME)

SCZ_SEARCH_NEAR_TIE = 1  # scz_info.search_flags: the device compared two costs within 1e-12


class _Info(ctypes.Structure):
    """scz_info (include/sczip_b200.h)."""

    _fields_ = [("status", ctypes.c_int32), ("version", ctypes.c_uint8),
                ("q_bits", ctypes.c_uint8), ("precision", ctypes.c_uint8),
                ("sym_bytes", ctypes.c_uint8), ("total", ctypes.c_uint64),
                ("n_rows", ctypes.c_uint32), ("n_cols", ctypes.c_uint32),
                ("nnz", ctypes.c_uint64), ("scale", ctypes.c_double),
                ("zero_point", ctypes.c_int64), ("alphabet", ctypes.c_uint32),
                ("lanes", ctypes.c_uint32), ("block_syms", ctypes.c_uint32),
                ("n_blocks", ctypes.c_uint32), ("payload_len", ctypes.c_uint64),
                ("payload_off", ctypes.c_uint64), ("freqs_off", ctypes.c_uint64),
                ("blocks_off", ctypes.c_uint64), ("search_flags", ctypes.c_uint32),
                ("n_evaluated", ctypes.c_uint32)]


_P = ctypes.c_void_p
_lib.scz_ctx_create.restype = ctypes.c_int
_lib.scz_ctx_create.argtypes = [ctypes.c_int, ctypes.POINTER(_P)]
_lib.scz_last_error.restype = ctypes.c_char_p          # a char*, not the default int
_lib.scz_last_error.argtypes = [_P]
_lib.scz_compress.restype = ctypes.c_int
_lib.scz_compress.argtypes = [_P, _P, ctypes.c_uint64, ctypes.c_int, ctypes.c_int64, ctypes.c_int, ctypes.c_int,
                              ctypes.c_uint32, ctypes.c_uint32, ctypes.POINTER(_Info),
                              ctypes.POINTER(ctypes.POINTER(ctypes.c_uint32)),
                              ctypes.POINTER(ctypes.POINTER(ctypes.c_uint32)),
                              ctypes.POINTER(ctypes.POINTER(ctypes.c_uint8))]
_lib.scz_decompress.restype = ctypes.c_int
_lib.scz_decompress.argtypes = [_P, ctypes.POINTER(_Info), _P, _P, _P, _P]

_ctx = _P()
if _lib.scz_ctx_create(0, ctypes.byref(_ctx)) != 0:
    raise ImportError("libsczip_b200: no sm_100 device")

# status code -> the reference exception class (errors.py:4-45)
_ERR = {1: "InvalidInput", 2: "NonDivisible", 3: "CorruptStream", 4: "InvalidContainer",
        5: "UnsupportedVersion", 6: "AlphabetOverflow", 7: "NormalizeError",
        8: "PrecisionTooSmall", 9: "UncodableSymbol"}


def _check(status: int) -> None:
    if status:
        msg = (_lib.scz_last_error(_ctx) or b"").decode(errors="replace")
        raise getattr(errors, _ERR.get(status, "SczipError"))(f"libsczip_b200 ({status}): {msg}")


def _run_compress(x: np.ndarray, q_bits: int, n_rows: int, precision: int):
    info = _Info()
    f = ctypes.POINTER(ctypes.c_uint32)()
    b = ctypes.POINTER(ctypes.c_uint32)()
    p = ctypes.POINTER(ctypes.c_uint8)()
    _check(_lib.scz_compress(_ctx, x.ctypes.data_as(_P), x.size, int(q_bits), int(n_rows), int(precision),
                             1, 32, 8192, ctypes.byref(info), ctypes.byref(f), ctypes.byref(b), ctypes.byref(p)))
    freqs = np.ctypeslib.as_array(f, shape=(info.alphabet,)).astype(np.int64)
    return info, freqs, ctypes.string_at(p, info.payload_len)


def compress(t: FeatureTensor, q_bits: int, n_rows=None, precision: int = 14) -> Container:
    """container.compress on the GPU, v1 wire format (the reference's bytes).

    The device prices every reshape candidate with CUDA's log2; when two
    compared costs are within 1e-12 relative (SCZ_SEARCH_NEAR_TIE) the last
    ulp of numpy's log2 decides, so N is re-decided here with the reference's
    own optimizer.search and the tensor re-coded if that differs.
    """
    x = np.ascontiguousarray(t.data, dtype=np.float32)
    info, freqs, payload = _run_compress(x, q_bits, -1 if n_rows is None else n_rows, precision)
    if n_rows is None and info.search_flags & SCZ_SEARCH_NEAR_TIE:
        n_host, _ = optimizer.search(t, q_bits)
        if n_host != info.n_rows:
            info, freqs, payload = _run_compress(x, q_bits, n_host, precision)
    return Container(q_bits=int(info.q_bits), precision=int(info.precision), dims=tuple(t.dims),
                     n_rows=int(info.n_rows), n_cols=int(info.n_cols), nnz=int(info.nnz),
                     scale=float(info.scale), zero_point=int(info.zero_point), freqs=freqs,
                     payload=payload)


def decompress(c: Container) -> FeatureTensor:
    """container.decompress on the GPU (v1 containers)."""
    if c.version != 1:
        raise errors.UnsupportedVersion(f"container version {c.version} unsupported")
    if c.n_rows * c.n_cols != c.total:
        raise errors.InvalidContainer("N * K does not match the product of dims")
    freqs = np.ascontiguousarray(c.freqs, dtype=np.int64)
    if int(freqs.sum()) != 1 << c.precision:
        raise errors.CorruptStream("frequencies do not sum to 2^precision")
    info = _Info(version=1, q_bits=c.q_bits & 0xFF, precision=c.precision & 0xFF, total=c.total,
                 n_rows=c.n_rows, n_cols=c.n_cols, nnz=c.nnz, scale=c.scale, zero_point=c.zero_point,
                 alphabet=freqs.size, lanes=1, block_syms=0, n_blocks=1, payload_len=len(c.payload))
    f32 = freqs.astype(np.uint32)
    payload = np.frombuffer(bytes(c.payload) or b"\0", np.uint8)
    out = np.empty(c.total, np.float32)
    _check(_lib.scz_decompress(_ctx, ctypes.byref(info), f32.ctypes.data_as(_P), None,
                               payload.ctypes.data_as(_P), out.ctypes.data_as(_P)))
    QuantParams(c.q_bits, c.scale, c.zero_point, 0.0, 0.0)  # container.py:120 order
    return FeatureTensor(c.dims, out)
