"""Reference containers of the general-alphabet cases (tests/inputs.py
GENERAL_ALPHABET: K > 65535, alphabets past 4096 / 8192), produced by the
UNMODIFIED reference (/root/reference/pkg/src, this container only):
sha256 of container.to_bytes(container.compress(t, q, n_rows, precision)) and
of decompress()'s float bits, written to tests/golden/general_alphabet.json.

Usage:  python tests/golden/make_golden_general.py
"""

import hashlib
import json
import os
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, "/root/reference/pkg/src")
sys.path.insert(0, os.path.dirname(HERE))

from sczip import container, tensor  # noqa: E402  (reference)

from inputs import GENERAL_ALPHABET, sparse_columns  # noqa: E402


def main():
    out = []
    for label, T, n_rows, stride, q, prec in GENERAL_ALPHABET:
        x = sparse_columns(T, T // n_rows, stride, seed=T % 997)
        t = tensor.FeatureTensor((T,), x)
        c = container.compress(t, q, n_rows, prec)
        raw = container.to_bytes(c)
        back = container.decompress(container.from_bytes(raw))
        out.append(dict(label=label, T=T, n_rows=n_rows, stride=stride, q=q, precision=prec,
                        input_sha=hashlib.sha256(x.tobytes()).hexdigest(),
                        alphabet=int(c.alphabet_size), bytes=len(raw),
                        container_sha=hashlib.sha256(raw).hexdigest(),
                        output_sha=hashlib.sha256(back.data.tobytes()).hexdigest()))
        print(label, out[-1]["alphabet"], out[-1]["bytes"], flush=True)
    with open(os.path.join(HERE, "general_alphabet.json"), "w") as f:
        json.dump(out, f, indent=1)


if __name__ == "__main__":
    main()
