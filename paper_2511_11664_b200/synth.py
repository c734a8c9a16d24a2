"""Synthetic feature tensors (the inputs of BASELINE.json's configs).

Restates the reference generator ``bench.gen_synthetic``
(/root/reference/pkg/src/sczip/bench.py:60-85) so parity tests and the bench
build bit-identical arrays without the reference present, plus the "signed"
distribution of SURVEY.md 8(d) (linear-bottleneck / hidden-state features).
"""

from __future__ import annotations

import numpy as np

from .errors import InvalidInput

KINDS = ("relu-laplace", "uniform", "constant")


def gen_synthetic_array(kind: str, dims, sparsity: float = 0.0, seed: int = 0) -> np.ndarray:
    """Flat float32 data of ``bench.gen_synthetic(kind, dims, sparsity, seed)``."""
    if kind not in KINDS:
        raise InvalidInput(f"unknown kind {kind!r}; choose from {KINDS}")
    if not 0.0 <= sparsity <= 1.0:
        raise InvalidInput(f"sparsity must be in [0, 1], got {sparsity}")
    total = int(np.prod(tuple(int(d) for d in dims)))
    rng = np.random.default_rng(seed)
    if kind == "constant":
        return np.ones(total, dtype=np.float32)
    if kind == "uniform":
        data = rng.random(total, dtype=np.float32)
        if sparsity > 0:
            data[rng.random(total) < sparsity] = 0.0
        return data
    data = np.abs(rng.laplace(0.0, 1.0, total)).astype(np.float32)
    data[rng.random(total) < sparsity] = 0.0
    return data


def signed_laplace(dims, seed: int = 0) -> np.ndarray:
    """Dense signed features: ``default_rng(seed).laplace(0, 1, T)`` as float32."""
    total = int(np.prod(tuple(int(d) for d in dims)))
    return np.random.default_rng(seed).laplace(0.0, 1.0, total).astype(np.float32)


def make_input(spec: dict) -> np.ndarray:
    """Input array for a golden/bench spec dict (kind, dims, sparsity, seed)."""
    kind, dims = spec["kind"], spec["dims"]
    total = int(np.prod(dims))
    if kind == "signed":
        return signed_laplace(dims, spec["seed"])
    if kind == "zeros":
        return np.zeros(total, np.float32)
    if kind == "single":
        return np.ones(total, np.float32)
    return gen_synthetic_array(kind, dims, spec.get("sparsity", 0.0), spec.get("seed", 0))
