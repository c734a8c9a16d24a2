"""Pin the CPU oracle (oracle/) to the unmodified reference.

The golden vectors were produced by tests/golden/make_golden.py importing
/root/reference/pkg/src/sczip; the KATs are the ones the reference's own
suite asserts (pkg/tests/test_rans.py, test_tensor.py, test_sparse.py).
CPU only -- these tests never need a GPU.
"""

import hashlib
import math
import os

import numpy as np
import pytest

from inputs import make_input
from oracle import oracle as orc

GOLDEN = os.path.join(os.path.dirname(__file__), "golden")


def sha(b):
    return hashlib.sha256(b).hexdigest()


# ---- known-answer tests copied from the reference's suite -----------------
def test_kat_compute_params():
    # test_tensor.py:19-45
    assert orc.compute_params(0.0, 255.0, 8) == (1.0, 0)
    assert orc.compute_params(0.0, 7.5, 4) == (0.5, 0)
    s, z = orc.compute_params(-1.0, 1.0, 2)
    assert s == pytest.approx(2 / 3) and z == 2
    assert orc.compute_params(0.0, 0.0, 4) == (1.0, 0)
    assert orc.compute_params(-3.0, -3.0, 4)[1] == 15
    for q in (1, 9, 0):
        with pytest.raises(orc.OracleError):
            orc.compute_params(0.0, 1.0, q)


def test_kat_quantize():
    # test_tensor.py:64-87
    q, m = orc.quantize(np.array([3.26], np.float32), 0.5, 0, 4)
    assert q[0] == 7 and not m[0]
    q, m = orc.quantize(np.array([0.0], np.float32), 0.5, 3, 4)
    assert q[0] == 3 and m[0]
    s, z = orc.compute_params(-1.0, 1.0, 2)
    q, _ = orc.quantize(np.array([1.0], np.float32), s, z, 2)
    assert q[0] == 3


def test_kat_normalize():
    # test_rans.py:52-76
    assert orc.normalize_frequencies([1, 2, 3, 1, 0, 1], 4).tolist() == [2, 4, 6, 2, 0, 2]
    assert orc.normalize_frequencies([7], 4).tolist() == [16]
    for counts, prec in (([1, 1, 1], 1), ([1] * 300, 8)):
        with pytest.raises(orc.OracleError) as e:
            orc.normalize_frequencies(counts, prec)
        assert e.value.status == orc.PRECISION_TOO_SMALL
    with pytest.raises(orc.OracleError) as e:
        orc.normalize_frequencies([0, 0, 0, 0], 10)
    assert e.value.status == orc.NORMALIZE_ERROR
    assert orc.normalize_frequencies([5, 0, 3], 8)[1] == 0


def test_kat_rans():
    # test_rans.py:101-125: zero-entropy stream is exactly the 4 state bytes
    f = orc.normalize_frequencies(orc.build_counts(np.zeros(50, np.uint32), 1), 14)
    b = orc.rans_encode(np.zeros(50, np.uint32), f, 14)
    assert len(b) == 4
    assert orc.rans_decode(b, f, 14, 50).tolist() == [0] * 50
    d = np.array([5, 3, 2, 1, 0, 2, 1, 2], np.uint32)
    f = orc.normalize_frequencies(orc.build_counts(d, 6), 14)
    assert orc.rans_decode(orc.rans_encode(d, f, 14), f, 14, 8).tolist() == d.tolist()
    # trailing garbage / truncation -> CorruptStream (test_rans.py:132-147)
    b = orc.rans_encode(d, f, 14)
    for bad in (b[:-1], b[:2], b + b"\x00"):
        with pytest.raises(orc.OracleError) as e:
            orc.rans_decode(bad, f, 14, 8)
        assert e.value.status == orc.CORRUPT_STREAM
    with pytest.raises(orc.OracleError) as e:
        orc.rans_encode(np.array([1], np.uint32), np.array([128, 0, 128]), 8)
    assert e.value.status == orc.UNCODABLE_SYMBOL
    with pytest.raises(orc.OracleError) as e:
        orc.rans_encode(np.array([2], np.uint32), np.array([128, 128]), 8)
    assert e.value.status == orc.ALPHABET_OVERFLOW


def test_kat_csr():
    # test_sparse.py:38-101
    q = np.array([0, 5, 0, 3, 0, 2], np.uint32)
    d, nnz = orc.csr_concat(q, q == 0, 2)
    assert nnz == 3 and d.tolist() == [5, 3, 2, 1, 0, 2, 1, 2]
    qq, m = orc.csr_decode(d, 3, 2, 3)
    assert qq.tolist() == q.tolist() and m.tolist() == (q == 0).tolist()
    for dd, nnz, n, k in (([1, 2, 3, 0, 1, 0, 2, 2], 3, 2, 3), ([1, 5, 1, 0], 1, 2, 3),
                          ([1, 2, 1, 1, 2, 0], 2, 2, 3)):
        with pytest.raises(orc.OracleError):
            orc.csr_decode(np.array(dd, np.uint32), nnz, n, k)


# ---- golden vectors from the unmodified reference -------------------------
def test_golden_quantize_and_params(golden):
    for row in golden["kat"]["quantize"]:
        x = np.array(row["x"], np.uint32).view(np.float32)
        s, z = orc.params_for(x, row["q"])
        assert s.hex() == row["scale"] and z == row["z"]
        q, m = orc.quantize(x, s, z, row["q"])
        assert q.tolist() == row["sym"] and m.tolist() == row["mask"]
        deq = orc.dequantize(q, m, s, z)
        assert deq.view(np.uint32).tolist() == row["deq"]
    for a, b, q, s_hex, z in golden["kat"]["params"]:
        s, zz = orc.compute_params(a, b, q)
        assert s.hex() == s_hex and zz == z


def test_golden_normalize(golden):
    for row in golden["kat"]["normalize"]:
        if isinstance(row["freqs"], str):
            with pytest.raises(orc.OracleError):
                orc.normalize_frequencies(row["counts"], row["precision"])
        else:
            assert orc.normalize_frequencies(row["counts"], row["precision"]).tolist() == row["freqs"]


def test_golden_rans_streams(golden):
    for row in golden["kat"]["rans"]:
        d = np.array(row["d"], np.uint32)
        counts = orc.build_counts(d, row["alphabet"])
        f = orc.normalize_frequencies(counts, row["precision"])
        assert f.tolist() == row["freqs"]
        b = orc.rans_encode(d, f, row["precision"])
        assert b.hex() == row["payload"]
        assert orc.rans_decode(b, f, row["precision"], d.size).tolist() == row["d"]


def _check_case(rec, full_bytes=None):
    spec = rec["spec"]
    x = make_input(spec)
    assert sha(x.tobytes()) == rec["input_sha"]
    q = spec["q"]
    if "search" in rec:
        n, cands, stopped = orc.search(x, q)
        want = rec["search"]
        assert n == want["chosen"] and stopped == want["early_stopped"]
        assert [list(c[:4]) for c in cands] == [c[:4] for c in want["candidates"]]
        for got, exp in zip(cands, want["candidates"]):
            assert got[4] == exp[4] and got[5] == exp[5]  # same numpy, same host
    c = orc.compress(x, spec["dims"], q, spec.get("n_rows"), spec.get("precision", 14))
    raw = orc.to_bytes(c)
    assert (c["n_rows"], c["nnz"], c["zero_point"]) == (rec["n_rows"], rec["nnz"], rec["zero_point"])
    assert sha(raw) == rec["container_sha"] and len(raw) == rec["container_len"]
    if full_bytes is not None:
        assert raw == full_bytes
    out = orc.decompress(c)
    assert sha(out.tobytes()) == rec["output_sha"]
    return x, c


def test_golden_small_containers(golden):
    for rec in golden["small"]:
        with open(os.path.join(GOLDEN, rec["file"]), "rb") as f:
            _check_case(rec, f.read())


def test_golden_exhaustive(golden):
    for rec in golden["small"] + golden["big"]:
        if "exhaustive" not in rec:
            continue
        x = make_input(rec["spec"])
        n, cands = orc.exhaustive_search(x, rec["spec"]["q"])
        assert n == rec["exhaustive"]["chosen"]
        assert [[c[0], c[4], c[5]] for c in cands] == rec["exhaustive"]["candidates"]


def test_golden_big_configs(golden):
    # BASELINE.json configs C1/C2/C5 (C4 too when generated with --big)
    for rec in golden["big"]:
        if rec["spec"].get("name") == "C4-llama2-7b":
            continue  # covered by test_golden_c4 (slow)
        _check_case(rec)


@pytest.mark.slow
def test_golden_c4(golden):
    for rec in golden["big"]:
        if rec["spec"].get("name") == "C4-llama2-7b":
            _check_case(rec)


def test_v2_lanes_equal_reference_encode(golden):
    """FORMAT.md v2: lane j of block b == rans.encode(D_block[j::W]) (reference)."""
    for rec in golden["small"] + golden["big"]:
        spec = rec["spec"]
        x = make_input(spec)
        s, z = orc.params_for(x, spec["q"])
        q, m = orc.quantize(x, s, z, spec["q"])
        d, nnz = orc.csr_concat(q, m, rec["n_rows"])
        f = orc.normalize_frequencies(orc.build_counts(d, int(d.max()) + 1),
                                      spec.get("precision", 14))
        pins = rec["v2_lane_pins"]
        W, B = pins["lanes"], pins["block_syms"]
        for b, j, h in pins["pins"]:
            sub = d[b * B:(b + 1) * B][j::W]
            assert sha(orc.rans_encode(sub, f, spec.get("precision", 14))) == h
        # and the interleaved container agrees with those lanes
        payload, bb = orc.rans_encode_v2(d, f, spec.get("precision", 14), W, B)
        assert int(bb.sum()) == len(payload)
        back = orc.rans_decode_v2(payload, bb, f, spec.get("precision", 14), d.size, W, B)
        assert np.array_equal(back, d)


def test_v2_single_lane_is_v1(golden):
    for rec in golden["small"]:
        with open(os.path.join(GOLDEN, rec["file"]), "rb") as f:
            raw = f.read()
        spec = rec["spec"]
        x = make_input(spec)
        c1 = orc.compress(x, spec["dims"], spec["q"], rec["n_rows"], spec.get("precision", 14))
        c2 = orc.compress(x, spec["dims"], spec["q"], rec["n_rows"], spec.get("precision", 14),
                          fmt=2, lanes=1, block_syms=1 << 30)
        assert c2["payload"] == c1["payload"]
        assert orc.to_bytes(c1) == raw


def test_oracle_self_round_trip_random():
    rng = np.random.default_rng(7)
    for _ in range(200):
        total = int(rng.integers(1, 700))
        divs = orc.divisors(total)
        n = int(divs[rng.integers(0, len(divs))])
        q = int(rng.integers(2, 9))
        x = np.abs(rng.laplace(0, 1, total)).astype(np.float32)
        x[rng.random(total) < rng.uniform(0, 1)] = 0
        for fmt in (1, 2):
            try:
                c = orc.compress(x, (total,), q, n, 14, fmt=fmt, lanes=4, block_syms=64)
            except orc.OracleError as e:
                assert e.status == orc.PRECISION_TOO_SMALL
                continue
            out = orc.decompress(c)
            s, z = orc.params_for(x, q)
            nz = x != 0
            assert np.all(out[~nz] == 0)
            if nz.any():
                assert np.abs(out[nz] - x[nz]).max() <= s + 1e-6


def test_oracle_general_alphabet_pinned_to_reference():
    """K > 65535 and alphabets past 4096 / 8192 (tests/inputs.py GENERAL_ALPHABET):
    the oracle's v1 containers and reconstructions equal the unmodified
    reference's (tests/golden/general_alphabet.json, make_golden_general.py)."""
    import hashlib
    import json

    from inputs import GENERAL_ALPHABET, sparse_columns

    pins = {r["label"]: r for r in json.load(open(os.path.join(GOLDEN, "general_alphabet.json")))}
    for label, T, n_rows, stride, q, prec in GENERAL_ALPHABET:
        x = sparse_columns(T, T // n_rows, stride, seed=T % 997)
        pin = pins[label]
        assert hashlib.sha256(x.tobytes()).hexdigest() == pin["input_sha"], label
        c = orc.compress(x, (T,), q, n_rows, prec)
        raw = orc.to_bytes(c)
        assert hashlib.sha256(raw).hexdigest() == pin["container_sha"], label
        assert hashlib.sha256(orc.decompress(c).tobytes()).hexdigest() == pin["output_sha"], label
