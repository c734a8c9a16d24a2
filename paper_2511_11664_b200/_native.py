"""ctypes binding of libsczip_b200.so (include/sczip_b200.h).

The product path has no CPU fallback: if the library is missing or no
sm_100 device is visible, every entry point raises ``DeviceError``.
"""

from __future__ import annotations

import ctypes
import os
import threading

import numpy as np

from .errors import STATUS_TO_ERROR, DeviceError

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(HERE, "_lib", "libsczip_b200.so")

SCZ_SEARCH_NEAR_TIE = 1
SCZ_SEARCH_EARLY_STOPPED = 2
SCZ_SEARCH_USED = 4


class Info(ctypes.Structure):
    """scz_info (include/sczip_b200.h)."""

    _fields_ = [
        ("status", ctypes.c_int32),
        ("version", ctypes.c_uint8),
        ("q_bits", ctypes.c_uint8),
        ("precision", ctypes.c_uint8),
        ("sym_bytes", ctypes.c_uint8),
        ("total", ctypes.c_uint64),
        ("n_rows", ctypes.c_uint32),
        ("n_cols", ctypes.c_uint32),
        ("nnz", ctypes.c_uint64),
        ("scale", ctypes.c_double),
        ("zero_point", ctypes.c_int64),
        ("alphabet", ctypes.c_uint32),
        ("lanes", ctypes.c_uint32),
        ("block_syms", ctypes.c_uint32),
        ("n_blocks", ctypes.c_uint32),
        ("payload_len", ctypes.c_uint64),
        ("payload_off", ctypes.c_uint64),
        ("freqs_off", ctypes.c_uint64),
        ("blocks_off", ctypes.c_uint64),
        ("search_flags", ctypes.c_uint32),
        ("n_evaluated", ctypes.c_uint32),
    ]


class Batch(ctypes.Structure):
    """scz_batch (include/sczip_b200.h)."""

    _fields_ = [
        ("batch", ctypes.c_uint32),
        ("d_info", ctypes.c_void_p),
        ("d_freqs", ctypes.c_void_p),
        ("d_block_bytes", ctypes.c_void_p),
        ("d_payload", ctypes.c_void_p),
        ("payload_total", ctypes.c_uint64),
        ("freqs_total", ctypes.c_uint64),
        ("blocks_total", ctypes.c_uint64),
    ]


INFO_DTYPE = np.dtype(
    [(name, {ctypes.c_int32: "<i4", ctypes.c_uint8: "u1", ctypes.c_uint32: "<u4",
             ctypes.c_uint64: "<u8", ctypes.c_double: "<f8", ctypes.c_int64: "<i8"}[t])
     for name, t in Info._fields_],
    align=True,
)
assert INFO_DTYPE.itemsize == ctypes.sizeof(Info)

EXPORTS = (
    "scz_abi_version", "scz_ctx_create", "scz_ctx_destroy", "scz_last_error", "scz_ctx_stream",
    "scz_launch_count", "scz_compress", "scz_decompress", "scz_encode_batch", "scz_batch_sync",
    "scz_decode_batch", "scz_decode_batch_async", "scz_decode_status", "scz_decode_batch_device", "scz_quantize",
    "scz_quantize_params", "scz_dequantize", "scz_csr_encode", "scz_csr_decode", "scz_build_counts",
    "scz_normalize", "scz_rans_encode", "scz_rans_decode", "scz_search", "scz_compress_batch",
    "scz_decompress_batch", "scz_ctx_set_timing", "scz_ctx_read_timing", "scz_last_call_ms",
    "scz_encode_batch_ptrs",
)

_lib = None
_lib_lock = threading.Lock()


def load_library():
    """Load libsczip_b200.so and declare its signatures (no device needed)."""
    global _lib
    with _lib_lock:
        if _lib is not None:
            return _lib
        if not os.path.exists(LIB_PATH):
            raise DeviceError(
                f"{LIB_PATH} is missing: build it with `python -c 'import __graft_entry__ as g; g.build()'`")
        lib = ctypes.CDLL(LIB_PATH)
        P, U32, U64, I32, I64, D = (ctypes.c_void_p, ctypes.c_uint32, ctypes.c_uint64,
                                    ctypes.c_int, ctypes.c_int64, ctypes.c_double)
        sig = {
            "scz_abi_version": (I32, []),
            "scz_ctx_create": (I32, [I32, P]),
            "scz_ctx_destroy": (None, [P]),
            "scz_last_error": (ctypes.c_char_p, [P]),
            "scz_ctx_stream": (P, [P]),
            "scz_launch_count": (U64, [P]),
            "scz_compress": (I32, [P, P, U64, I32, I64, I32, I32, U32, U32, P, P, P, P]),
            "scz_decompress": (I32, [P, P, P, P, P, P]),
            "scz_encode_batch": (I32, [P, P, U64, U32, I32, I64, I32, I32, U32, U32, P]),
            "scz_batch_sync": (I32, [P, P, P]),
            "scz_decode_batch": (I32, [P, P, U32, P, P, P, P, P]),
            "scz_decode_batch_async": (I32, [P, P, U32, P, P, P, P]),
            "scz_decode_status": (I32, [P, U32, P]),
            "scz_decode_batch_device": (I32, [P, P]),
            "scz_quantize": (I32, [P, P, U64, I32, P, P, P, P, P]),
            "scz_quantize_params": (I32, [P, P, U64, I32, D, I64, P, P]),
            "scz_dequantize": (I32, [P, P, P, U64, I32, D, I64, P]),
            "scz_csr_encode": (I32, [P, P, P, U64, U64, P, P]),
            "scz_csr_decode": (I32, [P, P, U64, U64, U64, P, P]),
            "scz_build_counts": (I32, [P, P, U64, U64, P]),
            "scz_normalize": (I32, [P, P, U64, I32, P]),
            "scz_rans_encode": (I32, [P, P, U64, P, U64, I32, U32, U32, P, P, P]),
            "scz_rans_decode": (I32, [P, P, U64, P, U64, I32, U32, U32, U64, P, U64, P]),
            "scz_search": (I32, [P, P, U64, I32, P, U32, U32, P, P, P, U32, P, P, P]),
            "scz_compress_batch": (I32, [P, P, U64, U32, I32, I64, I32, I32, U32, U32, P, P, P, P, P]),
            "scz_decompress_batch": (I32, [P, P, U32, P, U64, P, U64, P, U64, P, P]),
            "scz_ctx_set_timing": (I32, [P, I32]),
            "scz_ctx_read_timing": (I32, [P, ctypes.c_char_p, U64]),
            "scz_last_call_ms": (I32, [P, P]),
            "scz_encode_batch_ptrs": (I32, [P, P, P, U32, I32, I64, I32, I32, U32, U32, P]),
        }
        for name, (res, args) in sig.items():
            fn = getattr(lib, name)
            fn.restype = res
            fn.argtypes = args
        _lib = lib
        return lib


class Context:
    """One scz_ctx (CUDA stream + scratch) per thread and device."""

    def __init__(self, device: int = 0):
        lib = load_library()
        h = ctypes.c_void_p()
        st = lib.scz_ctx_create(int(device), ctypes.byref(h))
        if st != 0:
            raise DeviceError(
                f"scz_ctx_create(device={device}) failed with status {st}: "
                "no sm_100 CUDA device visible (the product has no CPU fallback)")
        self.lib = lib
        self.h = h
        self.device = device

    def __del__(self):
        h = getattr(self, "h", None)
        if h:
            try:
                self.lib.scz_ctx_destroy(h)
            except Exception:
                pass
            self.h = None

    def check(self, status: int, default_exc=None):
        if status == 0:
            return
        msg = (self.lib.scz_last_error(self.h) or b"").decode(errors="replace")
        exc = STATUS_TO_ERROR.get(status)
        if exc is None:
            raise DeviceError(f"libsczip_b200 status {status}: {msg}")
        raise exc(msg)

    @property
    def stream(self) -> int:
        return int(self.lib.scz_ctx_stream(self.h) or 0)

    @property
    def launches(self) -> int:
        return int(self.lib.scz_launch_count(self.h))

    def last_call_ms(self) -> float:
        """CUDA-event device time of the last host-buffer call (scz_last_call_ms)."""
        ms = ctypes.c_float()
        self.check(self.lib.scz_last_call_ms(self.h, ctypes.byref(ms)))
        return float(ms.value)

    def set_timing(self, enable: bool) -> None:
        self.check(self.lib.scz_ctx_set_timing(self.h, 1 if enable else 0))

    def read_timing(self) -> dict[str, tuple[float, int]]:
        """{kernel: (total ms, launches)} since the last read (CUDA events)."""
        buf = ctypes.create_string_buffer(1 << 16)
        self.check(self.lib.scz_ctx_read_timing(self.h, buf, len(buf)))
        out = {}
        for line in buf.value.decode().splitlines():
            name, ms, n = line.split()
            out[name] = (float(ms), int(n))
        return out


_tls = threading.local()


def context(device: int | None = None) -> Context:
    """The calling thread's context for `device` (default: current torch/CUDA device 0)."""
    dev = 0 if device is None else int(device)
    cache = getattr(_tls, "ctx", None)
    if cache is None:
        cache = _tls.ctx = {}
    ctx = cache.get(dev)
    if ctx is None:
        ctx = cache[dev] = Context(dev)
    return ctx


def ptr(a: np.ndarray):
    return a.ctypes.data_as(ctypes.c_void_p)
