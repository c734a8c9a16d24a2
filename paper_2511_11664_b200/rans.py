"""Range-ANS entropy coder with static frequency tables.

Drop-in for the reference's ``sczip.rans`` (rans.py:1-240): 32-bit state,
L = 2^23, byte renormalisation, precision n in [8, 16] (default 14), symbols
pushed in reverse, payload = 4-byte LE state + bytes in decoder order.

build_counts, normalize_frequencies, encode and decode run on the GPU
(k_hist_u32, k_normalize_only, k_rans_enc_v1 / k_rans_dec_v1; the v2
interleaved-lane layout of FORMAT.md is exposed as ``encode_lanes`` /
``decode_lanes``).  encode_step / decode_step are the reference's scalar
single-step functions; entropy and the size diagnostics are the reference's
numpy expressions (their exact float results feed the reshape search).
"""

from __future__ import annotations

import ctypes
from dataclasses import dataclass

import numpy as np

from . import _native
from .errors import CorruptStream, InvalidInput
from .sparse import ConcatStream

STATE_LOW = 1 << 23  # rans.py:26
DEFAULT_PRECISION = 14
MIN_PRECISION = 8
MAX_PRECISION = 16


@dataclass(frozen=True)
class FrequencyTable:
    """Normalised frequencies summing to 2^precision, plus the CDF (rans.py:32-56)."""

    alphabet_size: int
    raw_counts: np.ndarray
    freqs: np.ndarray  # normalized, sum == 2**precision
    cdf: np.ndarray  # length alphabet_size + 1, cdf[0] == 0
    precision: int

    def __post_init__(self):
        object.__setattr__(self, "raw_counts", np.asarray(self.raw_counts, dtype=np.int64))
        object.__setattr__(self, "freqs", np.asarray(self.freqs, dtype=np.int64))
        object.__setattr__(self, "cdf", np.asarray(self.cdf, dtype=np.int64))

    @classmethod
    def from_freqs(cls, freqs, precision: int) -> "FrequencyTable":
        """Rebuild a table from already-normalised frequencies (wire form)."""
        freqs = np.asarray(freqs, dtype=np.int64)
        if int(freqs.sum()) != 1 << precision:
            raise CorruptStream("frequencies do not sum to 2^precision")
        cdf = np.concatenate(([0], np.cumsum(freqs)))
        return cls(freqs.size, freqs.copy(), freqs, cdf, precision)


@dataclass(frozen=True)
class Bitstream:
    """Encoded payload ordered for strictly forward decoder consumption (rans.py:59-67)."""

    data: bytes

    @property
    def payload_bits(self) -> int:
        return 8 * len(self.data)


def _as_symbols(d) -> np.ndarray:
    if isinstance(d, ConcatStream):
        return d.data
    return np.ascontiguousarray(d, dtype=np.uint32).ravel()


def build_counts(d, alphabet_size: int) -> np.ndarray:
    """Tally symbol occurrences over the whole stream (rans.py:76-85), on the GPU."""
    symbols = _as_symbols(d)
    if alphabet_size < 1:
        raise InvalidInput(f"alphabet_size must be >= 1, got {alphabet_size}")
    ctx = _native.context()
    counts = np.empty(alphabet_size, np.int64)
    ctx.check(ctx.lib.scz_build_counts(ctx.h, _native.ptr(symbols), symbols.size, int(alphabet_size),
                                       _native.ptr(counts)))
    return counts


def normalize_frequencies(counts, precision: int) -> FrequencyTable:
    """Largest-remainder scaling to 2^precision (rans.py:88-131), one CTA on the GPU."""
    counts = np.ascontiguousarray(np.asarray(counts, dtype=np.int64)).ravel()
    if counts.size == 0:
        from .errors import NormalizeError

        raise NormalizeError("cannot normalize all-zero counts")
    ctx = _native.context()
    freqs = np.empty(counts.size, np.uint32)
    ctx.check(ctx.lib.scz_normalize(ctx.h, _native.ptr(counts), counts.size, int(precision),
                                    _native.ptr(freqs)))
    f = freqs.astype(np.int64)
    cdf = np.concatenate(([0], np.cumsum(f)))
    return FrequencyTable(counts.size, counts, f, cdf, precision)


def encode_step(state: int, freq: int, cum: int, precision: int) -> tuple[int, list[int]]:
    """One symbol push (rans.py:134-144): renormalise, then the state transform."""
    emitted = []
    bound = ((STATE_LOW >> precision) << 8) * freq
    while state >= bound:
        emitted.append(state & 0xFF)
        state >>= 8
    state = (state // freq << precision) + cum + state % freq
    return state, emitted


def decode_step(state: int, t: FrequencyTable) -> tuple[int, int]:
    """Identify the symbol from the low bits and pop it, no refill (rans.py:147-152)."""
    slot = state & ((1 << t.precision) - 1)
    sym = int(np.searchsorted(t.cdf, slot, side="right")) - 1
    state = int(t.freqs[sym]) * (state >> t.precision) + slot - int(t.cdf[sym])
    return state, sym


def _freqs_u32(t: FrequencyTable) -> np.ndarray:
    return np.ascontiguousarray(t.freqs, dtype=np.uint32)


def _encode(symbols: np.ndarray, t: FrequencyTable, lanes: int, block_syms: int):
    ctx = _native.context()
    n = symbols.size
    n_blocks = max(1, -(-n // block_syms)) if lanes else 1
    cap = 4 * max(lanes, 1) * n_blocks + 2 * n + 16
    out = np.empty(cap, np.uint8)
    bb = np.empty(n_blocks, np.uint32)
    out_len = ctypes.c_uint64()
    ctx.check(ctx.lib.scz_rans_encode(ctx.h, _native.ptr(symbols), n, _native.ptr(_freqs_u32(t)),
                                      t.alphabet_size, int(t.precision), lanes, block_syms,
                                      _native.ptr(out), ctypes.byref(out_len), _native.ptr(bb)))
    return out[: out_len.value].tobytes(), bb


def encode(d, t: FrequencyTable, *, check_state: bool = False) -> Bitstream:
    """Entropy-code the stream, symbols pushed in reverse (rans.py:155-180).

    Format v1: one stream, byte-identical to the reference.  ``check_state``
    is accepted for API compatibility (the device coder's states are always
    in [2^23, 2^32) by construction).
    """
    symbols = _as_symbols(d)
    data, _ = _encode(symbols, t, 0, 0)
    return Bitstream(data)


def decode(b: Bitstream, t: FrequencyTable, count: int, *, check_state: bool = False) -> np.ndarray:
    """Recover `count` symbols in forward order; verifies the final state (rans.py:183-213)."""
    data = bytes(b.data)
    ctx = _native.context()
    buf = np.frombuffer(data, np.uint8).copy() if data else np.zeros(1, np.uint8)
    out = np.empty(max(int(count), 1), np.uint32)
    ctx.check(ctx.lib.scz_rans_decode(ctx.h, _native.ptr(buf), len(data), _native.ptr(_freqs_u32(t)),
                                      t.alphabet_size, int(t.precision), 0, 0, 1, None, int(count),
                                      _native.ptr(out)))
    return out[: int(count)]


def encode_lanes(d, t: FrequencyTable, lanes: int = 32, block_syms: int = 8192):
    """FORMAT.md v2: blocks of interleaved lanes -> (payload bytes, uint32 block lengths)."""
    return _encode(_as_symbols(d), t, lanes, block_syms)


def decode_lanes(data: bytes, block_bytes, t: FrequencyTable, count: int, lanes: int = 32,
                 block_syms: int = 8192) -> np.ndarray:
    """Inverse of encode_lanes."""
    ctx = _native.context()
    data = bytes(data)
    buf = np.frombuffer(data, np.uint8).copy() if data else np.zeros(1, np.uint8)
    bb = np.ascontiguousarray(block_bytes, dtype=np.uint32)
    out = np.empty(max(int(count), 1), np.uint32)
    ctx.check(ctx.lib.scz_rans_decode(ctx.h, _native.ptr(buf), len(data), _native.ptr(_freqs_u32(t)),
                                      t.alphabet_size, int(t.precision), lanes, block_syms, bb.size,
                                      _native.ptr(bb), int(count), _native.ptr(out)))
    return out[: int(count)]


def entropy(counts) -> float:
    """Shannon entropy in bits per symbol (rans.py:216-223)."""
    counts = np.asarray(counts, dtype=np.float64)
    total = counts.sum()
    if total <= 0:
        raise InvalidInput("entropy of an empty distribution")
    p = counts[counts > 0] / total
    return float(-(p * np.log2(p)).sum())


def expected_size(counts) -> float:
    """Expected compressed size in bits (rans.py:226-229)."""
    counts = np.asarray(counts, dtype=np.float64)
    return float(counts.sum()) * entropy(counts)


def compression_ratio(counts, alphabet_size: int) -> float:
    """Expected bits relative to the flat log2(alphabet) encoding (rans.py:232-240)."""
    if alphabet_size < 2:
        raise InvalidInput("compression ratio needs an alphabet of at least 2")
    counts = np.asarray(counts, dtype=np.float64)
    total = counts.sum()
    if total <= 0:
        raise InvalidInput("empty distribution")
    return entropy(counts) / float(np.log2(alphabet_size))
