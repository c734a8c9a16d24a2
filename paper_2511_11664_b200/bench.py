"""Synthetic activations (the reference's ``sczip.bench.gen_synthetic``).

bench.py:60-85 of the reference; the timing sweep of that module is a
"next" row of SURVEY.md 8(f) and lives in the repo-root bench.py harness.
"""

from __future__ import annotations

from .synth import KINDS, gen_synthetic_array
from .tensor import FeatureTensor


def gen_synthetic(kind: str, dims, sparsity: float = 0.0, seed: int = 0) -> FeatureTensor:
    """Deterministic stand-in activations (bench.py:60-85)."""
    dims = tuple(int(d) for d in dims)
    return FeatureTensor(dims, gen_synthetic_array(kind, dims, sparsity, seed))


__all__ = ["KINDS", "gen_synthetic"]
