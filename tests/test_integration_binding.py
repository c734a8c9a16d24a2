"""Executes the reference-side binding of INTEGRATION.md
(integration/sczip_b200_binding.py) as a maintainer would install it: as
module ``sczip._b200`` inside a package named ``sczip``.  The drop-in package
stands in for the reference here (the reference is absent on the GPU box);
the binding only uses the names both packages share (errors, optimizer,
container.Container, tensor.FeatureTensor / QuantParams)."""

import importlib.util
import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
BINDING = os.path.join(ROOT, "integration", "sczip_b200_binding.py")
LIB = os.path.join(ROOT, "paper_2511_11664_b200", "_lib", "libsczip_b200.so")

# Runs in a subprocess: the alias `sczip` -> paper_2511_11664_b200 and the
# SCZ_FORCE_NEAR_TIE switch must not leak into other tests.
SCRIPT = r'''
import importlib.util, os, sys, json
import numpy as np
sys.path.insert(0, {root!r}); sys.path.insert(0, os.path.join({root!r}, "tests"))
import paper_2511_11664_b200 as pkg
from paper_2511_11664_b200 import container, errors, optimizer, tensor
sys.modules["sczip"] = pkg
for name in ("container", "errors", "optimizer", "tensor", "rans", "sparse"):
    sys.modules["sczip." + name] = getattr(pkg, name)
spec = importlib.util.spec_from_file_location("sczip._b200", {binding!r})
b200 = importlib.util.module_from_spec(spec)
sys.modules["sczip._b200"] = b200
spec.loader.exec_module(b200)

golden = json.load(open(os.path.join({root!r}, "tests", "golden", "golden.json")))
from inputs import make_input
n = 0
for rec in golden["small"]:
    spec_ = rec["spec"]
    t = tensor.FeatureTensor(tuple(spec_["dims"]), make_input(spec_))
    c = b200.compress(t, spec_["q"], spec_.get("n_rows"), spec_.get("precision", 14))
    want = open(os.path.join({root!r}, "tests", "golden", rec["file"]), "rb").read()
    assert container.to_bytes(c) == want, spec_
    out = b200.decompress(container.from_bytes(want))
    assert np.array_equal(out.data.view(np.uint32), pkg.decompress(container.from_bytes(want)).data.view(np.uint32))
    n += 1
# errors surface as the reference classes with the library's message (scz_last_error as char*)
t = tensor.FeatureTensor((8, 8, 8), make_input(dict(kind="relu-laplace", dims=[8, 8, 8], sparsity=0.8, seed=21)))
try:
    b200.compress(t, 4, 7)
    raise SystemExit("no error")
except errors.NonDivisible as e:
    assert "divide" in str(e), e
bad = container.from_bytes(container.to_bytes(b200.compress(t, 4)))
bad = container.Container(bad.q_bits, bad.precision, bad.dims, bad.n_rows, bad.n_cols, bad.nnz, bad.scale,
                          bad.zero_point, bad.freqs, bad.payload[:-1])
try:
    b200.decompress(bad)
    raise SystemExit("no error")
except errors.CorruptStream:
    pass
# near ties: with SCZ_FORCE_NEAR_TIE every searched tensor is flagged; the
# binding re-decides with optimizer.search and re-codes when N differs
if os.environ.get("SCZ_FORCE_NEAR_TIE"):
    t = pkg.gen_synthetic("relu-laplace", [1, 64, 28, 28], 0.5, 3)
    c0 = b200.compress(t, 8)
    assert container.to_bytes(c0) == container.to_bytes(pkg.compress(t, 8))
    calls = []
    real = optimizer.search
    def fake(t_, q_):
        calls.append(q_)
        return 1568, None                       # another feasible N (K = 32)
    optimizer.search = fake
    c1 = b200.compress(t, 8)
    optimizer.search = real
    assert calls and c1.n_rows == 1568
    assert container.to_bytes(c1) == container.to_bytes(pkg.compress(t, 8, 1568))
print("binding ok", n)
'''


def _run(extra_env):
    env = dict(os.environ, SCZIP_B200_LIB=LIB, **extra_env)
    code = SCRIPT.format(root=ROOT, binding=BINDING)
    return subprocess.run([sys.executable, "-c", code], env=env, capture_output=True, text=True, timeout=600)


@pytest.mark.gpu
@pytest.mark.parametrize("tie", [False, True])
def test_reference_binding_round_trips_golden_containers(tie):
    out = _run({"SCZ_FORCE_NEAR_TIE": "1"} if tie else {})
    assert out.returncode == 0 and "binding ok" in out.stdout, out.stdout[-2000:] + out.stderr[-4000:]


def test_binding_declares_every_symbol_it_calls():
    """CPU check: every scz_* function the binding calls has its restype and
    argtypes declared (an undeclared char* restype truncates the pointer)."""
    src = open(BINDING).read()
    import re

    called = set(re.findall(r"_lib\.(scz_\w+)\(", src))
    for name in called:
        assert f"_lib.{name}.restype" in src and f"_lib.{name}.argtypes" in src, name
    assert "_lib.scz_last_error.restype = ctypes.c_char_p" in src
    spec = importlib.util.spec_from_file_location("binding_syntax", BINDING)
    assert spec is not None
    compile(src, BINDING, "exec")
