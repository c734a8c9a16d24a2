"""Test-side access to the synthetic input generator (see synth.py)."""

import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

from paper_2511_11664_b200.synth import make_input  # noqa: E402,F401


def sparse_columns(T, K, stride, seed):
    """Nonzeros only in every `stride`-th column of the N x K view (plus the
    last column), so the column alphabet reaches K while the number of
    distinct symbols stays within 2^precision (general-alphabet cases)."""
    import numpy as np

    rng = np.random.default_rng(seed)
    x = np.zeros(T, np.float32)
    cols = np.arange(T) % K
    keep = (cols % stride == 0) | (cols == K - 1)
    keep &= rng.random(T) < 0.6
    x[keep] = np.abs(rng.laplace(0, 1, int(keep.sum()))).astype(np.float32) + 0.01
    return x


# (label, T, n_rows, stride, q, precision): K = T / n_rows.  Reference
# containers of these are pinned in tests/golden/general_alphabet.json.
GENERAL_ALPHABET = [
    ("u32-K131072", 131072 * 3, 3, 8, 8, 14),       # K > 65535: u32 symbols, A > 8192, binary-search decode
    ("u16-K10000", 1_000_000, 100, 1, 8, 15),       # A > 8192 (global encoder tables), u16 symbols
    ("u16-K3000", 3000 * 64, 64, 1, 6, 14),         # 4096 >= A > 256: u16 LUT decode
    ("u16-K40000-sparse", 40000 * 5, 5, 4, 4, 14),  # A ~ 40000 > 2^14 slots with ~10k distinct symbols
]
