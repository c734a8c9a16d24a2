"""CPU-side checks of the boundary: the C-ABI library loads and exports every
entry point include/sczip_b200.h declares, the host-only header code matches
the reference wire format, and the product refuses to run without a device
(no CPU fallback)."""

import ctypes
import os
import re

import numpy as np
import pytest

from paper_2511_11664_b200 import _native, container, errors, optimizer

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "sczip_b200.h")
GOLDEN = os.path.join(ROOT, "tests", "golden")


def declared_functions():
    text = open(HEADER).read()
    return sorted(set(re.findall(r"^\s*(?:int|void|const char\*|void\*|uint64_t)\s+\*?(scz_\w+)\(",
                                 text, re.M)))


def test_header_declares_entry_points():
    names = declared_functions()
    assert "scz_compress" in names and "scz_decompress" in names and len(names) >= 20
    assert set(names) == set(_native.EXPORTS)


def test_library_exports_every_declared_symbol():
    lib = _native.load_library()
    for name in declared_functions():
        assert hasattr(lib, name), name
    assert lib.scz_abi_version() == 1


def test_info_struct_layout_matches_header(tmp_path):
    """The ctypes mirror of scz_info / scz_batch has the C compiler's layout."""
    import subprocess

    fields = [f for f, _ in _native.Info._fields_]
    src = tmp_path / "layout.c"
    src.write_text(
        "#include <stdio.h>\n#include <stddef.h>\n#include \"sczip_b200.h\"\nint main(void){\n"
        + 'printf("%zu %zu\\n", sizeof(scz_info), sizeof(scz_batch));\n'
        + "".join(f'printf("%zu\\n", offsetof(scz_info, {f}));\n' for f in fields)
        + "return 0;}\n")
    exe = tmp_path / "layout"
    subprocess.check_call(["gcc", "-I", os.path.join(ROOT, "include"), "-o", str(exe), str(src)])
    out = subprocess.check_output([str(exe)], text=True).split()
    assert int(out[0]) == ctypes.sizeof(_native.Info)
    assert int(out[1]) == ctypes.sizeof(_native.Batch)
    for f, off in zip(fields, out[2:]):
        assert getattr(_native.Info, f).offset == int(off), f


def test_no_cpu_fallback_without_device():
    import torch

    if torch.cuda.is_available():
        pytest.skip("a GPU is present")
    with pytest.raises(errors.DeviceError):
        _native.Context(0)


def test_status_codes_map_to_reference_classes():
    want = {1: "InvalidInput", 2: "NonDivisible", 3: "CorruptStream", 4: "InvalidContainer",
            5: "UnsupportedVersion", 6: "AlphabetOverflow", 7: "NormalizeError",
            8: "PrecisionTooSmall", 9: "UncodableSymbol"}
    for code, name in want.items():
        assert errors.STATUS_TO_ERROR[code].__name__ == name
    text = open(HEADER).read()
    for code, name in want.items():
        assert re.search(rf"= {code},\s*/\* errors\.{name} \*/", text), name


def test_wire_format_round_trip_on_reference_containers(golden):
    """from_bytes/to_bytes (host) reproduce the reference's v1 bytes exactly."""
    for rec in golden["small"]:
        raw = open(os.path.join(GOLDEN, rec["file"]), "rb").read()
        c = container.from_bytes(raw)
        assert container.to_bytes(c) == raw
        assert c.total_bytes == len(raw) == rec["container_len"]
        assert (c.n_rows, c.n_cols, c.nnz) == (rec["n_rows"], rec["n_cols"], rec["nnz"])


def test_header_error_classes_match_reference(golden):
    """Header-level corruption raises what the reference's from_bytes raises."""
    for case in golden["errors"]:
        blob = bytes.fromhex(case["blob"])
        try:
            c = container.from_bytes(blob)
        except (errors.SczipError, ValueError) as e:
            assert type(e).__name__ == case["error"], case["name"]
            continue
        # parsed fine: the remaining failures are raised by decompress (GPU tests)
        assert case["error"] in (None, "CorruptStream", "InvalidInput", "InvalidContainer"), case


def test_candidate_rows_match_reference_rule():
    from oracle import oracle as orc

    for total in (1, 2, 16, 36, 100, 360, 100352, 401408, 802816, 150528, 12544):
        for q in range(2, 9):
            assert optimizer.candidate_rows(total, q) == orc.candidate_rows(total, q)


def test_encoder_reciprocal_is_exact():
    """floor(x / f) == umulhi(x, m) >> (l - 1) for the encoder's state range
    (x < 2^31), every f in [2, 2^16] at boundary x values."""
    f = np.arange(2, (1 << 16) + 1, dtype=np.uint64)
    l = np.array([(int(v) - 1).bit_length() for v in f], dtype=np.uint64)  # ceil(log2 f)
    m = ((np.uint64(1) << (np.uint64(31) + l)) + f - np.uint64(1)) // f
    assert int(m.max()) < (1 << 32)
    rng = np.random.default_rng(0)
    for xs in ([0, 1, (1 << 31) - 1, (1 << 23), (1 << 30)],
               rng.integers(0, 1 << 31, 64).tolist()):
        for x0 in xs:
            x = np.full(f.shape, x0, dtype=np.uint64)
            q = ((x * m) >> np.uint64(32)) >> (l - np.uint64(1))
            assert np.array_equal(q, x // f)
        # values just below / at multiples of f
        k = rng.integers(1, 1 << 15, f.shape).astype(np.uint64)
        for delta in (0, 1):
            x = np.minimum(k * f - np.uint64(delta), np.uint64((1 << 31) - 1))
            q = ((x * m) >> np.uint64(32)) >> (l - np.uint64(1))
            assert np.array_equal(q, x // f)
