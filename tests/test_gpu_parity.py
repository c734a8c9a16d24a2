"""GPU parity: the sm_100a path through the C-ABI against the reference's
golden bytes and the CPU oracle (bit-exact for every integer / byte output,
0-ulp for the fp32 reconstruction).  Mirrors the reference's own suite
(pkg/tests/test_*.py) where it asserts known answers."""

import hashlib
import os

import numpy as np
import pytest

import paper_2511_11664_b200 as sz
from inputs import make_input
from oracle import oracle as orc
from paper_2511_11664_b200 import container, optimizer, rans, sparse, tensor
from paper_2511_11664_b200.errors import (
    AlphabetOverflow,
    CorruptStream,
    InvalidContainer,
    InvalidInput,
    NonDivisible,
    NormalizeError,
    PrecisionTooSmall,
    UncodableSymbol,
    UnsupportedVersion,
)

pytestmark = pytest.mark.gpu
GOLDEN = os.path.join(os.path.dirname(__file__), "golden")


def sha(b):
    return hashlib.sha256(b).hexdigest()


def tensor_of(spec):
    return sz.FeatureTensor(tuple(spec["dims"]), make_input(spec))


# ------------------------------------------------------------ containers
def test_v1_containers_bit_exact_vs_reference_files(golden):
    """compress() reproduces the reference's .scz bytes; decompress() its floats."""
    for rec in golden["small"]:
        spec = rec["spec"]
        t = tensor_of(spec)
        c = sz.compress(t, spec["q"], spec.get("n_rows"), spec.get("precision", 14))
        raw = container.to_bytes(c)
        want = open(os.path.join(GOLDEN, rec["file"]), "rb").read()
        assert raw == want, spec
        out = sz.decompress(container.from_bytes(want))
        assert sha(out.data.tobytes()) == rec["output_sha"], spec


def test_v1_baseline_configs_bit_exact(golden):
    """BASELINE.json configs C1, C2 (VGG16, MobileNetV2), C5 (SwinT, DenseNet, Q=2..8)."""
    for rec in golden["big"]:
        spec = rec["spec"]
        if spec.get("name") == "C4-llama2-7b":
            continue
        t = tensor_of(spec)
        c = sz.compress(t, spec["q"])
        assert c.n_rows == rec["n_rows"], spec["name"]
        raw = container.to_bytes(c)
        assert sha(raw) == rec["container_sha"], spec["name"]
        out = sz.decompress(c)
        assert sha(out.data.tobytes()) == rec["output_sha"], spec["name"]


def test_v1_llama_hidden_state_c4(golden):
    """C4: 1x2048x4096 signed dense, K=1, l_D = 25.2M symbols in one v1 stream."""
    rec = next((r for r in golden["big"] if r["spec"].get("name") == "C4-llama2-7b"), None)
    if rec is None:
        pytest.skip("golden.json generated without --big")
    t = tensor_of(rec["spec"])
    c = sz.compress(t, 8, format=2)
    assert c.n_rows == rec["n_rows"] and c.nnz == rec["nnz"]
    out = sz.decompress(c)
    assert sha(out.data.tobytes()) == rec["output_sha"]
    c1 = sz.compress(t, 8)
    assert sha(container.to_bytes(c1)) == rec["container_sha"]


def test_v2_containers_match_oracle(golden):
    for rec in golden["small"] + golden["big"]:
        spec = rec["spec"]
        if spec.get("name") == "C4-llama2-7b":
            continue
        t = tensor_of(spec)
        for bs in (64, 8192):
            c = sz.compress(t, spec["q"], spec.get("n_rows"), spec.get("precision", 14),
                            format=2, block_syms=bs)
            ref = orc.compress(t.data, t.dims, spec["q"], rec["n_rows"], spec.get("precision", 14),
                               fmt=2, lanes=32, block_syms=bs)
            assert container.to_bytes(c) == orc.to_bytes(ref), (spec, bs)
            back = container.from_bytes(container.to_bytes(c))
            out = sz.decompress(back)
            assert sha(out.data.tobytes()) == rec["output_sha"], (spec, bs)


def test_v2_lanes_are_reference_streams(golden):
    """Each lane of a v2 block is exactly rans.encode of its subsequence (reference pins)."""
    for rec in golden["big"][:3]:
        spec = rec["spec"]
        t = tensor_of(spec)
        pins = rec["v2_lane_pins"]
        W, B = pins["lanes"], pins["block_syms"]
        p = tensor.params_for(t, spec["q"])
        q = tensor.quantize_reshape(t, p, rec["n_rows"])
        d = sparse.concat(sparse.csr_encode(q))
        table = rans.normalize_frequencies(rans.build_counts(d, int(d.data.max()) + 1), 14)
        for b, j, h in pins["pins"]:
            sub = d.data[b * B:(b + 1) * B][j::W]
            assert sha(rans.encode(sub, table).data) == h


# ----------------------------------------------------------- stage parity
def test_quantize_kat_and_edge_values(golden):
    for row in golden["kat"]["quantize"]:
        x = np.array(row["x"], np.uint32).view(np.float32)
        t = sz.FeatureTensor((x.size,), x)
        p = tensor.params_for(t, row["q"])
        assert p.scale.hex() == row["scale"] and p.zero_point == row["z"]
        q, m = tensor.quantize(t, p)
        assert q.tolist() == row["sym"] and m.tolist() == row["mask"]
        out = tensor.dequantize(sz.QuantizedMatrix(1, x.size, q, m), p, (x.size,))
        assert out.data.view(np.uint32).tolist() == row["deq"]
    # test_tensor.py:64-87
    q, m = tensor.quantize(sz.FeatureTensor((1,), np.array([3.26], np.float32)),
                           sz.QuantParams(4, 0.5, 0, 0.0, 7.5))
    assert q[0] == 7 and not m[0]
    q, m = tensor.quantize(sz.FeatureTensor((1,), np.array([0.0], np.float32)),
                           sz.QuantParams(4, 0.5, 3, -1.5, 6.0))
    assert q[0] == 3 and m[0]
    vals = np.array([-1e6, -0.8, 0.0, 0.7, 1e6], np.float32)
    q, _ = tensor.quantize(sz.FeatureTensor((5,), vals), sz.QuantParams(4, 0.1, 8, -0.8, 0.7))
    assert q.max() <= 15


def test_quantize_matches_oracle_random():
    """fp32 guard band + fp64 fix-up == the reference's fp64 sequence, incl.
    values planted on and one ulp around every rounding boundary."""
    rng = np.random.default_rng(1)
    for trial in range(24):
        q_bits = 2 + trial % 7
        n = int(rng.integers(1, 300_000))
        x = (rng.laplace(0, 1, n) * rng.choice([1e-3, 1, 1e3])).astype(np.float32)
        if trial % 3 == 0:
            x = np.abs(x)
        x[rng.random(n) < 0.3] = 0.0
        x[rng.random(n) < 0.01] = -0.0
        s, z = orc.params_for(x, q_bits)
        k = rng.integers(0, (1 << q_bits) - 1, min(n, 5000))
        planted = ((k + 0.5 - z) * s).astype(np.float32)
        idx = rng.integers(0, n, planted.size)
        x[idx] = np.nextafter(planted, planted + rng.choice([-1, 0, 1], planted.size).astype(np.float32))
        t = sz.FeatureTensor((n,), x)
        p = tensor.params_for(t, q_bits)
        s, z = orc.params_for(x, q_bits)
        assert (p.scale, p.zero_point) == (s, z)
        q, m = tensor.quantize(t, p)
        qo, mo = orc.quantize(x, s, z, q_bits)
        assert np.array_equal(q, qo) and np.array_equal(m, mo)
        out = tensor.dequantize(sz.QuantizedMatrix(1, n, q, m), p, (n,))
        assert np.array_equal(out.data.view(np.uint32), orc.dequantize(qo, mo, s, z).view(np.uint32))


def test_pipeline_guard_band_planted_boundaries():
    """The batch pipeline's quantiser (unclamped magic-constant symbols, 2^-13
    guard band, deferred fp64 path) against the oracle on tensors whose
    values sit on and one ulp around rounding boundaries: v1 containers
    byte-identical, v2 containers identical to the oracle's."""
    rng = np.random.default_rng(11)
    for trial in range(6):
        q_bits = (8, 4, 2, 6, 8, 3)[trial]
        n = 96 * 1024
        x = (rng.laplace(0, 1, n) * (1e-2, 1.0, 300.0)[trial % 3]).astype(np.float32)
        if trial % 2 == 0:
            x = np.abs(x)  # post-ReLU: z = 0
        x[rng.random(n) < 0.4] = 0.0
        s, z = orc.params_for(x, q_bits)
        k = rng.integers(0, (1 << q_bits) - 1, 20000)
        planted = ((k + 0.5 - z) * s).astype(np.float32)
        lo, hi = x.min(), x.max()
        planted = np.clip(planted, lo, hi)  # keep the tensor's range (and params)
        idx = rng.integers(0, n, planted.size)
        x[idx] = np.nextafter(planted, planted + rng.choice([-1, 0, 1], planted.size).astype(np.float32))
        t = sz.FeatureTensor((n,), x)
        for fmt in (1, 2):
            c = sz.compress(t, q_bits, format=fmt)
            ref = orc.compress(x, (n,), q_bits, None if fmt == 1 else c.n_rows, fmt=fmt)
            assert container.to_bytes(c) == orc.to_bytes(ref), (trial, fmt)


def test_csr_kat_and_corruption():
    # test_sparse.py:38-101
    q = sz.QuantizedMatrix(2, 3, [0, 5, 0, 3, 0, 2], [True, False, True, False, True, False])
    s = sparse.csr_encode(q)
    assert s.values.tolist() == [5, 3, 2] and s.col_idx.tolist() == [1, 0, 2]
    assert s.row_counts.tolist() == [1, 2]
    back = sparse.csr_decode(s, 2, 3)
    assert back.data.tolist() == [0, 5, 0, 3, 0, 2]
    assert back.zero_mask.tolist() == [True, False, True, False, True, False]
    e = sparse.csr_encode(sz.QuantizedMatrix(2, 3, np.zeros(6), np.ones(6, bool)))
    assert e.values.size == 0 and e.row_counts.tolist() == [0, 0]
    assert sparse.csr_encode(sz.QuantizedMatrix(1, 2, [0, 3], [False, False])).values.tolist() == [0, 3]
    for bad in (sz.SparseCSR([1, 2, 3], [0, 1, 0], [2, 2]), sz.SparseCSR([1], [5], [1, 0]),
                sz.SparseCSR([1, 2], [1, 1], [2, 0]), sz.SparseCSR([1], [0], [1])):
        with pytest.raises(CorruptStream):
            sparse.csr_decode(bad, 2, 3)


def test_csr_matches_oracle_random():
    rng = np.random.default_rng(2)
    for _ in range(40):
        n, k = int(rng.integers(1, 400)), int(rng.integers(1, 300))
        qv = rng.integers(0, 256, n * k).astype(np.uint32)
        mask = rng.random(n * k) < rng.uniform(0, 1)
        s = sparse.csr_encode(sz.QuantizedMatrix(n, k, qv, mask))
        d, nnz = orc.csr_concat(qv, mask, n)
        assert np.array_equal(sparse.concat(s).data, d)
        back = sparse.csr_decode(s, n, k)
        qo, mo = orc.csr_decode(d, nnz, n, k)
        assert np.array_equal(back.data, qo) and np.array_equal(back.zero_mask, mo)


def test_counts_and_normalize(golden):
    assert rans.build_counts([5, 3, 2, 1, 0, 2, 1, 2], 6).tolist() == [1, 2, 3, 1, 0, 1]
    assert rans.build_counts([], 4).tolist() == [0, 0, 0, 0]
    with pytest.raises(AlphabetOverflow):
        rans.build_counts([0, 7], 6)
    t = rans.normalize_frequencies([1, 2, 3, 1, 0, 1], 4)
    assert t.freqs.tolist() == [2, 4, 6, 2, 0, 2] and t.cdf.tolist() == [0, 2, 6, 12, 14, 14, 16]
    assert rans.normalize_frequencies([7], 4).freqs.tolist() == [16]
    with pytest.raises(PrecisionTooSmall):
        rans.normalize_frequencies([1, 1, 1], 1)
    with pytest.raises(PrecisionTooSmall):
        rans.normalize_frequencies([1] * 300, 8)
    with pytest.raises(NormalizeError):
        rans.normalize_frequencies([0, 0, 0, 0], 10)
    for row in golden["kat"]["normalize"]:
        if isinstance(row["freqs"], str):
            with pytest.raises(PrecisionTooSmall):
                rans.normalize_frequencies(row["counts"], row["precision"])
        else:
            got = rans.normalize_frequencies(row["counts"], row["precision"]).freqs.tolist()
            assert got == row["freqs"]
    rng = np.random.default_rng(3)
    for _ in range(200):
        a = int(rng.integers(1, 3000))
        counts = rng.integers(0, 2000, a) ** int(rng.integers(1, 3))
        counts[rng.random(a) < 0.3] = 0
        if counts.sum() == 0:
            continue
        prec = int(rng.integers(8, 17))
        try:
            want = orc.normalize_frequencies(counts, prec).tolist()
        except orc.OracleError:
            with pytest.raises(PrecisionTooSmall):
                rans.normalize_frequencies(counts, prec)
            continue
        assert rans.normalize_frequencies(counts, prec).freqs.tolist() == want


def test_rans_streams_match_reference(golden):
    for row in golden["kat"]["rans"]:
        d = np.array(row["d"], np.uint32)
        t = rans.FrequencyTable.from_freqs(row["freqs"], row["precision"])
        b = rans.encode(d, t)
        assert b.data.hex() == row["payload"]
        assert rans.decode(b, t, d.size).tolist() == row["d"]


def test_rans_kat_and_errors():
    # test_rans.py:101-157
    assert rans.encode_step(8388608, freq=6, cum=10, precision=4) == (22369628, [])
    t = rans.FrequencyTable.from_freqs([10, 6], 4)
    assert rans.decode_step(22369628, t) == (8388608, 1)
    d = [0] * 50
    t = rans.normalize_frequencies(rans.build_counts(d, 1), 14)
    b = rans.encode(d, t)
    assert len(b.data) == 4 and rans.decode(b, t, 50).tolist() == d
    t0 = rans.FrequencyTable.from_freqs([256], 8)
    assert rans.decode(rans.encode([], t0), t0, 0).size == 0
    rng = np.random.default_rng(0)
    d = rng.integers(0, 16, 500)
    t = rans.normalize_frequencies(rans.build_counts(d, 16), 14)
    b = rans.encode(d, t)
    for bad in (b.data[:-1], b.data[:2], b.data + b"\x00"):
        with pytest.raises(CorruptStream):
            rans.decode(rans.Bitstream(bad), t, 500)
    with pytest.raises(UncodableSymbol):
        rans.encode([1], rans.FrequencyTable.from_freqs([128, 0, 128], 8))
    with pytest.raises(AlphabetOverflow):
        rans.encode([2], rans.FrequencyTable.from_freqs([128, 128], 8))


def test_rans_random_vs_oracle_all_precisions():
    rng = np.random.default_rng(4)
    for trial in range(60):
        prec = 8 + trial % 9
        a = int(rng.integers(1, 300 if trial % 5 else 5000))
        n = int(rng.integers(1, 40_000))
        w = rng.random(a) ** 3
        d = rng.choice(a, size=n, p=w / w.sum()).astype(np.uint32)
        counts = np.bincount(d, minlength=a)
        try:
            f = orc.normalize_frequencies(counts, prec)
        except orc.OracleError:
            continue
        t = rans.FrequencyTable.from_freqs(f, prec)
        b = rans.encode(d, t)
        assert b.data == orc.rans_encode(d, f, prec)
        assert np.array_equal(rans.decode(b, t, n), d)
        if prec <= 16:
            payload, bb = rans.encode_lanes(d, t, 32, 32 * (1 + trial % 9))
            want, wbb = orc.rans_encode_v2(d, f, prec, 32, 32 * (1 + trial % 9))
            assert payload == want and bb.tolist() == wbb.tolist()
            back = rans.decode_lanes(payload, bb, t, n, 32, 32 * (1 + trial % 9))
            assert np.array_equal(back, d)


def test_search_reports_match_reference(golden):
    """optimizer.search / exhaustive_search: same N, candidates and entropy floats."""
    for rec in golden["small"] + golden["big"]:
        if "search" not in rec:
            continue
        t = tensor_of(rec["spec"])
        n, rep = optimizer.search(t, rec["spec"]["q"])
        want = rec["search"]
        assert n == want["chosen"] and rep.early_stopped == want["early_stopped"]
        got = [[c.n_rows, c.n_cols, c.nnz, c.stream_len, c.entropy_bits, c.t_tot]
               for c in rep.candidates]
        assert got == want["candidates"], rec["spec"]
        if "exhaustive" in rec:
            n, rep = optimizer.exhaustive_search(t, rec["spec"]["q"])
            assert n == rec["exhaustive"]["chosen"]
            assert [[c.n_rows, c.entropy_bits, c.t_tot] for c in rep.candidates] == \
                rec["exhaustive"]["candidates"]


def test_cost_on_infeasible_reshapes():
    # test_optimizer.py:58-63 trend + explicit N outside the search window
    t = sz.gen_synthetic("relu-laplace", [128, 28, 28], 0.9, 42)
    ent = [optimizer.cost(t, n, 4).entropy_bits for n in (784, 1792, 6272, 14336)]
    assert all(a > b for a, b in zip(ent, ent[1:]))
    x = t.data
    s, z = orc.params_for(x, 4)
    q, m = orc.quantize(x, s, z, 4)
    for n in (784, 1792, 6272, 14336):
        counts, _ = orc.stream_counts(q, m, n, 4)
        assert optimizer.cost(t, n, 4).entropy_bits == orc.entropy(counts)
    with pytest.raises(NonDivisible):
        optimizer.cost(sz.gen_synthetic("uniform", [4, 4], 0.0, 0), 5, 4)


def test_device_search_decision_matches_reference(golden):
    """The compress() path decides N on the device (fp64 entropy, numpy
    summation order); it must agree with the reference's choice."""
    for rec in golden["small"] + golden["big"]:
        if "search" not in rec or rec["spec"].get("name") == "C4-llama2-7b":
            continue
        rows, chosen, chosen_ex, flags = optimizer.device_histograms(tensor_of(rec["spec"]),
                                                                     rec["spec"]["q"])
        assert rows[chosen][0] == rec["search"]["chosen"], rec["spec"]


# ------------------------------------------------------------ error paths
def test_container_error_classes(golden):
    for case in golden["errors"]:
        blob = bytes.fromhex(case["blob"])
        try:
            container.decompress(container.from_bytes(blob))
            got = None
        except (sz.SczipError, ValueError) as e:
            got = type(e).__name__
        assert got == case["error"], case["name"]


def test_compress_argument_errors():
    t = sz.gen_synthetic("relu-laplace", [8, 8, 8], 0.8, 21)
    with pytest.raises(NonDivisible):
        sz.compress(t, 4, n_rows=7)
    with pytest.raises(InvalidInput):
        sz.compress(t, 4, precision=16)
    with pytest.raises(InvalidInput):
        sz.compress(t, 9)
    c = sz.compress(t, 4)
    bad = container.Container(c.q_bits, c.precision, c.dims, c.n_rows, c.n_cols + 1, c.nnz,
                              c.scale, c.zero_point, c.freqs, c.payload)
    with pytest.raises(InvalidContainer):
        sz.decompress(bad)
    bad = container.Container(c.q_bits, c.precision, c.dims, c.n_rows, c.n_cols, c.nnz,
                              c.scale, c.zero_point, c.freqs, c.payload[:-2])
    with pytest.raises(CorruptStream):
        sz.decompress(bad)
    with pytest.raises(UnsupportedVersion):
        sz.decompress(container.Container(c.q_bits, c.precision, c.dims, c.n_rows, c.n_cols,
                                          c.nnz, c.scale, c.zero_point, c.freqs, c.payload, 7))


def test_v2_corruption_detected():
    t = sz.gen_synthetic("relu-laplace", [1, 64, 28, 28], 0.5, 3)
    c = sz.compress(t, 8, format=2, block_syms=1024)
    raw = bytearray(container.to_bytes(c))
    for pos in (len(raw) - 1, len(raw) - 700, len(raw) - 3000):
        bad = bytearray(raw)
        bad[pos] ^= 0x5A
        with pytest.raises(CorruptStream):
            container.decompress(container.from_bytes(bytes(bad)))


# ------------------------------------------------------- random round trips
def test_random_round_trips_vs_oracle():
    """Acceptance-style (test_acceptance.py:44-62): random (T, Q, N), both formats."""
    rng = np.random.default_rng(7)
    for i in range(120):
        total = int(rng.integers(1, 5000))
        divs = orc.divisors(total)
        n_rows = None if i % 3 == 0 else int(divs[rng.integers(0, len(divs))])
        q = int(rng.integers(2, 9))
        x = np.abs(rng.laplace(0, 1, total)).astype(np.float32)
        x[rng.random(total) < rng.uniform(0.0, 0.97)] = 0.0
        if i % 7 == 0:
            x = -x
        t = sz.FeatureTensor((total,), x)
        fmt = 1 + i % 2
        try:
            ref = orc.compress(x, (total,), q, n_rows, 14, fmt=fmt, lanes=32, block_syms=256)
        except orc.OracleError as e:
            assert e.status == orc.PRECISION_TOO_SMALL
            with pytest.raises(PrecisionTooSmall):
                sz.compress(t, q, n_rows, format=fmt, block_syms=256)
            continue
        c = sz.compress(t, q, n_rows, format=fmt, block_syms=256)
        assert container.to_bytes(c) == orc.to_bytes(ref), (i, total, q, n_rows, fmt)
        out = sz.decompress(c)
        assert np.array_equal(out.data.view(np.uint32), orc.decompress(ref).view(np.uint32))


def test_precisions_round_trip_vs_oracle():
    """Every rANS precision of the container API (container.py:80-84: 8..15),
    both formats, on tensors long enough that the v1 coders' queues and
    payload-window rings wrap many times (tens of thousands of symbols)."""
    rng = np.random.default_rng(11)
    for i, precision in enumerate(range(8, 16)):
        for fmt in (1, 2):
            total = int(rng.integers(20000, 90000))
            q = int(rng.integers(4, 9))
            x = rng.laplace(0, 1, total).astype(np.float32)
            if i % 2 == 0:
                x = np.abs(x)
                x[rng.random(total) < 0.5] = 0.0
            t = sz.FeatureTensor((total,), x)
            try:
                ref = orc.compress(x, (total,), q, None, precision, fmt=fmt, lanes=32, block_syms=2048)
            except orc.OracleError as e:
                assert e.status == orc.PRECISION_TOO_SMALL
                with pytest.raises(PrecisionTooSmall):
                    sz.compress(t, q, None, precision=precision, format=fmt, block_syms=2048)
                continue
            c = sz.compress(t, q, None, precision=precision, format=fmt, block_syms=2048)
            assert container.to_bytes(c) == orc.to_bytes(ref), (precision, fmt, total, q)
            out = sz.decompress(c)
            assert np.array_equal(out.data.view(np.uint32), orc.decompress(ref).view(np.uint32))


def test_corrupt_payload_outcomes_match_oracle():
    """Bit flips and byte replacements anywhere in the payload of v1 and v2
    containers: the GPU decoders and the oracle reach the same outcome -- the same error class
    (rans.py:199-212 underrun / final-state / leftover-byte checks, the row
    checks of sparse.py:84-97) or bit-identical output."""
    from paper_2511_11664_b200.errors import STATUS_TO_ERROR, SczipError

    rng = np.random.default_rng(13)
    total = 40000
    x = np.abs(rng.laplace(0, 1, total)).astype(np.float32)
    x[rng.random(total) < 0.5] = 0.0
    t = sz.FeatureTensor((total,), x)
    for fmt in (1, 2):
        ref = orc.compress(x, (total,), 8, None, 14, fmt=fmt, lanes=32, block_syms=2048)
        raw = container.to_bytes(sz.compress(t, 8, None, format=fmt, block_syms=2048))
        assert raw == orc.to_bytes(ref)
        plen = len(ref["payload"])
        for k in range(64):
            # 48 single-bit flips, then 16 whole-byte replacements
            pos = int(rng.integers(0, plen))
            bit = 1 << int(rng.integers(0, 8)) if k < 48 else int(rng.integers(1, 256))
            bad = bytearray(raw)
            bad[len(raw) - plen + pos] ^= bit
            pl = bytearray(ref["payload"])
            pl[pos] ^= bit
            try:
                want, werr = orc.decompress(dict(ref, payload=bytes(pl))), None
            except orc.OracleError as e:
                want, werr = None, STATUS_TO_ERROR[e.status]
            try:
                got, gerr = sz.decompress(container.from_bytes(bytes(bad))).data, None
            except SczipError as e:
                got, gerr = None, type(e)
            assert gerr is werr, (fmt, pos, bit, gerr, werr)
            if werr is None:
                assert np.array_equal(got.view(np.uint32), want.view(np.uint32)), (fmt, pos, bit)


def test_corrupt_block_table_outcomes_match_oracle():
    """v2 block-length tables edited with the total kept (so the container
    still parses): lengths swapped, bytes moved between neighbours, a block
    shorter than its 32 lane states.  GPU decode and oracle agree on the
    error class or on bit-identical output."""
    import dataclasses

    from paper_2511_11664_b200.errors import STATUS_TO_ERROR, SczipError

    rng = np.random.default_rng(17)
    total = 60000
    x = rng.laplace(0, 1, total).astype(np.float32)
    t = sz.FeatureTensor((total,), x)
    ref = orc.compress(x, (total,), 8, None, 14, fmt=2, lanes=32, block_syms=2048)
    c = sz.compress(t, 8, None, format=2, block_syms=2048)
    assert container.to_bytes(c) == orc.to_bytes(ref)
    bb0 = np.asarray(ref["block_bytes"], dtype=np.int64)
    nb = bb0.size
    assert nb >= 4
    cases = []
    for _ in range(12):
        i = int(rng.integers(0, nb - 1))
        kind = int(rng.integers(0, 3))
        bb = bb0.copy()
        if kind == 0:
            bb[i], bb[i + 1] = bb[i + 1], bb[i]
        elif kind == 1:
            d = int(rng.integers(1, 5)) * (1 if rng.random() < 0.5 else -1)
            bb[i] += d
            bb[i + 1] -= d
        else:
            d = int(bb[i]) - 100  # shorter than the 128 state bytes
            bb[i] -= d
            bb[i + 1] += d
        cases.append(bb)
    for bb in cases:
        if (bb <= 0).any():
            continue
        try:
            want, werr = orc.decompress(dict(ref, block_bytes=bb.astype(np.uint32))), None
        except orc.OracleError as e:
            want, werr = None, STATUS_TO_ERROR[e.status]
        try:
            got, gerr = sz.decompress(dataclasses.replace(c, block_bytes=bb.astype(np.uint32))).data, None
        except SczipError as e:
            got, gerr = None, type(e)
        assert gerr is werr, (bb.tolist()[:6], gerr, werr)
        if werr is None:
            assert np.array_equal(got.view(np.uint32), want.view(np.uint32))


def test_batch_decode_isolates_corrupt_tensors():
    """One batch decode (scz_decompress_batch) over good and corrupted v1 / v2
    containers: every corrupted tensor reports the oracle's status, every good
    tensor decodes bit-identically -- a bad stream never leaks into its
    neighbours (per-tensor status)."""
    import ctypes

    from paper_2511_11664_b200 import _native

    rng = np.random.default_rng(19)
    conts, refs = [], []
    for i in range(10):
        total = int(rng.integers(5000, 30000))
        x = np.abs(rng.laplace(0, 1, total)).astype(np.float32)
        x[rng.random(total) < 0.5] = 0.0
        fmt = 1 + i % 2
        ref = orc.compress(x, (total,), 8, None, 14, fmt=fmt, lanes=32, block_syms=2048)
        c = sz.compress(sz.FeatureTensor((total,), x), 8, None, format=fmt, block_syms=2048)
        if i in (2, 5, 6):  # corrupt these: flip a payload byte
            pos = int(rng.integers(4, len(ref["payload"])))
            pl = bytearray(ref["payload"])
            pl[pos] ^= 0x5A
            ref = dict(ref, payload=bytes(pl))
            raw = bytearray(container.to_bytes(c))
            raw[len(raw) - len(pl) + pos] ^= 0x5A
            c = container.from_bytes(bytes(raw))
        conts.append(c)
        refs.append(ref)
    B = len(conts)
    infos = (_native.Info * B)()
    pay_off = fr_off = bl_off = 0
    for i, c in enumerate(conts):
        info = container._info_for(c)
        info.payload_off, info.freqs_off, info.blocks_off = pay_off, fr_off, bl_off
        infos[i] = info
        pay_off += len(c.payload)
        fr_off += c.alphabet_size
        bl_off += c.n_blocks if c.version == 2 else 0
    payload = np.frombuffer(b"".join(bytes(c.payload) for c in conts), np.uint8)
    freqs = np.concatenate([np.asarray(c.freqs, dtype=np.uint32) for c in conts])
    blocks = np.concatenate([np.asarray(c.block_bytes, dtype=np.uint32) for c in conts if c.version == 2])
    out = np.empty(sum(c.total for c in conts), np.float32)
    status = (ctypes.c_int32 * B)()
    ctx = _native.context()
    ctx.check(ctx.lib.scz_decompress_batch(ctx.h, infos, B, _native.ptr(freqs), freqs.size, _native.ptr(blocks),
                                           bl_off, _native.ptr(payload), pay_off, _native.ptr(out), status))
    pos = 0
    for i, (c, ref) in enumerate(zip(conts, refs)):
        try:
            want, wst = orc.decompress(ref), 0
        except orc.OracleError as e:
            want, wst = None, e.status
        assert int(status[i]) == wst, (i, int(status[i]), wst)
        if wst == 0:
            assert np.array_equal(out[pos: pos + c.total].view(np.uint32), want.view(np.uint32)), i
        pos += c.total


def test_edge_tensors_batch_vs_oracle():
    """Degenerate and extreme tensors through one batch encode / decode
    (compress_many / decompress_many) in both formats: all zeros, one
    nonzero, a constant (hi == lo: scale 1.0), signed with -0.0 entries,
    subnormal magnitudes and magnitudes near the fp32 maximum (both outside
    the fp32 guard-band range: the exact fp64 path for every element), one
    element.  Containers byte-identical to the oracle, outputs bit-identical."""
    T = 4096
    rng = np.random.default_rng(23)
    base = np.abs(rng.laplace(0, 1, T)).astype(np.float32)
    cases = {
        "zeros": np.zeros(T, np.float32),
        "one_nonzero": np.where(np.arange(T) == 1234, np.float32(3.5), np.float32(0.0)).astype(np.float32),
        "constant": np.full(T, 0.75, np.float32),
        "signed_negzero": np.where(rng.random(T) < 0.3, np.float32(-0.0),
                                   rng.laplace(0, 1, T).astype(np.float32)).astype(np.float32),
        "subnormal": (base * np.float32(1e-41)).astype(np.float32),
        "huge": (base / base.max() * np.float32(3e38)).astype(np.float32),
    }
    for fmt in (1, 2):
        for q in (2, 8):
            names = list(cases)
            ts = [sz.FeatureTensor((T,), cases[n]) for n in names]
            got = container.compress_many(ts, q, None, format=fmt, block_syms=2048)
            for n, c in zip(names, got):
                ref = orc.compress(cases[n], (T,), q, None, 14, fmt=fmt, lanes=32, block_syms=2048)
                assert container.to_bytes(c) == orc.to_bytes(ref), (n, fmt, q)
            outs = container.decompress_many(got)
            for n, o, c in zip(names, outs, got):
                ref = orc.compress(cases[n], (T,), q, None, 14, fmt=fmt, lanes=32, block_syms=2048)
                assert np.array_equal(o.data.view(np.uint32), orc.decompress(ref).view(np.uint32)), (n, fmt, q)
        # a one-element tensor on the single-tensor path
        one = np.array([1.25], np.float32)
        c = sz.compress(sz.FeatureTensor((1,), one), 8, None, format=fmt, block_syms=2048)
        ref = orc.compress(one, (1,), 8, None, 14, fmt=fmt, lanes=32, block_syms=2048)
        assert container.to_bytes(c) == orc.to_bytes(ref), fmt
        assert np.array_equal(sz.decompress(c).data.view(np.uint32), orc.decompress(ref).view(np.uint32))


def test_concurrent_threads_match_oracle():
    """Four host threads, each with its own library context (thread-local,
    _native.context), compress and decompress different tensors at the same
    time in both formats and through the batch API: every container and
    reconstruction equals the oracle's (contexts share no mutable state)."""
    import threading

    rng = np.random.default_rng(29)
    work = []
    for k in range(4):
        xs = []
        for j in range(3):
            total = int(rng.integers(3000, 20000))
            x = np.abs(rng.laplace(0, 1, total)).astype(np.float32)
            x[rng.random(total) < 0.5] = 0.0
            xs.append(x)
        work.append(xs)
    want = [[(orc.to_bytes(orc.compress(x, (x.size,), 8, None, 14, fmt=f, lanes=32, block_syms=2048)))
             for x in xs for f in (1, 2)] for xs in work]
    errors = []

    def run(k):
        try:
            for _ in range(4):
                got = []
                for x in work[k]:
                    for f in (1, 2):
                        c = sz.compress(sz.FeatureTensor((x.size,), x), 8, None, format=f, block_syms=2048)
                        got.append(container.to_bytes(c))
                        out = sz.decompress(c)
                        ref = orc.compress(x, (x.size,), 8, None, 14, fmt=f, lanes=32, block_syms=2048)
                        assert np.array_equal(out.data.view(np.uint32), orc.decompress(ref).view(np.uint32))
                assert got == want[k], k
                many = container.compress_many([sz.FeatureTensor((x.size,), x) for x in work[k]], 8, None,
                                               format=2, block_syms=2048)
                assert [container.to_bytes(c) for c in many] == want[k][1::2], k
        except Exception as e:  # surfaced below
            errors.append((k, e))

    th = [threading.Thread(target=run, args=(k,)) for k in range(4)]
    for t in th:
        t.start()
    for t in th:
        t.join()
    assert not errors, errors


def test_context_recovers_after_errors():
    """Failing calls leave the calling thread's context usable: corrupt
    containers (single and batch decode), invalid arguments and a
    NonDivisible reshape, each followed by a good round trip on the same
    context (graph caches included), which must still equal the oracle."""
    rng = np.random.default_rng(31)
    total = 24000
    x = np.abs(rng.laplace(0, 1, total)).astype(np.float32)
    x[rng.random(total) < 0.5] = 0.0
    t = sz.FeatureTensor((total,), x)
    refs = {f: orc.compress(x, (total,), 8, None, 14, fmt=f, lanes=32, block_syms=2048) for f in (1, 2)}
    good = {f: sz.compress(t, 8, None, format=f, block_syms=2048) for f in (1, 2)}

    def check_good():
        for f in (1, 2):
            c = sz.compress(t, 8, None, format=f, block_syms=2048)
            assert container.to_bytes(c) == orc.to_bytes(refs[f])
            assert np.array_equal(sz.decompress(c).data.view(np.uint32),
                                  orc.decompress(refs[f]).view(np.uint32))
        outs = container.decompress_many([good[1], good[2]])
        for o, f in zip(outs, (1, 2)):
            assert np.array_equal(o.data.view(np.uint32), orc.decompress(refs[f]).view(np.uint32))

    for it in range(3):
        for f in (1, 2):
            raw = bytearray(container.to_bytes(good[f]))
            raw[-5] ^= 0xFF  # a payload byte near the end
            bad = container.from_bytes(bytes(raw))
            try:
                sz.decompress(bad)
            except CorruptStream:
                pass
            try:
                container.decompress_many([good[1], bad, good[2]])
            except CorruptStream:
                pass
            check_good()
        with pytest.raises(NonDivisible):
            sz.compress(t, 8, 7)  # 7 does not divide 24000
        with pytest.raises(InvalidInput):
            sz.compress(t, 0)
        check_good()


def test_random_mixed_batches_vs_oracle():
    """Randomised batches through compress_many / decompress_many: tensors of
    different sizes (heterogeneous batch encode), sparsities and signs, the
    search on, one Q per batch, both formats, odd block sizes."""
    rng = np.random.default_rng(37)
    for it in range(6):
        q = int(rng.integers(2, 9))
        fmt = 1 + it % 2
        bs = int(rng.choice([256, 1024, 4096]))
        xs = []
        for _ in range(int(rng.integers(5, 14))):
            total = int(rng.integers(100, 30000))
            x = rng.laplace(0, 1, total).astype(np.float32)
            if rng.random() < 0.6:
                x = np.abs(x)
                x[rng.random(total) < rng.uniform(0.0, 0.95)] = 0.0
            xs.append(x)
        ts = [sz.FeatureTensor((x.size,), x) for x in xs]
        got = container.compress_many(ts, q, None, format=fmt, block_syms=bs)
        outs = container.decompress_many(got)
        for x, c, o in zip(xs, got, outs):
            ref = orc.compress(x, (x.size,), q, None, 14, fmt=fmt, lanes=32, block_syms=bs)
            assert container.to_bytes(c) == orc.to_bytes(ref), (it, x.size, q, fmt)
            assert np.array_equal(o.data.view(np.uint32), orc.decompress(ref).view(np.uint32)), (it, x.size)


def test_batch_api_matches_single_tensor_path():
    """compress_many / decompress_many (one device pass) == per-tensor calls."""
    ts = [sz.gen_synthetic("relu-laplace", [1, 64, 28, 28], 0.5 + 0.05 * i, 100 + i) for i in range(9)]
    for fmt in (1, 2):
        many = container.compress_many(ts, 8, format=fmt, block_syms=1024)
        for t, c in zip(ts, many):
            one = sz.compress(t, 8, format=fmt, block_syms=1024)
            assert container.to_bytes(c) == container.to_bytes(one)
        outs = container.decompress_many(many)
        for t, c, o in zip(ts, many, outs):
            assert np.array_equal(o.data.view(np.uint32), sz.decompress(c).data.view(np.uint32))
    # explicit N, mixed corruption: the bad tensor raises, as decompress would
    many = container.compress_many(ts[:3], 6, n_rows=50176 // 8, format=2, block_syms=512)
    assert all(c.n_cols == 8 for c in many)


def test_graph_replay_tracks_new_inputs_and_reallocation():
    """Repeated shapes replay a captured CUDA graph: every replay must see the
    new input values (device) and new headers (decode), and a buffer
    reallocation in between (a larger tensor) must invalidate the graphs."""
    rng = np.random.default_rng(11)
    shapes = [(1, 32, 20, 20)] * 4 + [(1, 64, 56, 56)] + [(1, 32, 20, 20)] * 4
    for i, dims in enumerate(shapes):
        t = sz.gen_synthetic("relu-laplace", list(dims), float(rng.uniform(0.3, 0.9)), 1000 + i)
        for fmt in (1, 2):
            ref = orc.compress(t.data, dims, 6, None, 14, fmt=fmt, lanes=32, block_syms=2048)
            c = sz.compress(t, 6, format=fmt, block_syms=2048)
            assert container.to_bytes(c) == orc.to_bytes(ref), (i, fmt)
            out = sz.decompress(c)
            assert np.array_equal(out.data.view(np.uint32), orc.decompress(ref).view(np.uint32)), (i, fmt)


def test_chunked_host_batch_calls(tmp_path):
    """compress_many / decompress_many split large batches into chunks whose
    copies overlap the kernels; with tiny chunks forced (SCZ_CHUNK_BYTES) the
    containers and reconstructions equal the single-tensor path."""
    import subprocess
    import sys

    code = (
        "import sys; sys.path.insert(0, %r); import numpy as np; import paper_2511_11664_b200 as sz\n"
        "from paper_2511_11664_b200 import container\n"
        "ts = [sz.gen_synthetic('relu-laplace', [1, 32, 28, 28], 0.3 + 0.02 * i, 50 + i) for i in range(19)]\n"
        "for fmt in (1, 2):\n"
        "    many = container.compress_many(ts, 8, format=fmt, block_syms=2048)\n"
        "    for t, c in zip(ts, many):\n"
        "        assert container.to_bytes(c) == container.to_bytes(sz.compress(t, 8, format=fmt, block_syms=2048))\n"
        "    outs = container.decompress_many(many)\n"
        "    for c, o in zip(many, outs):\n"
        "        assert np.array_equal(o.data.view(np.uint32), sz.decompress(c).data.view(np.uint32))\n"
        "print('ok')\n"
    )
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    env = dict(os.environ)
    env["SCZ_CHUNK_BYTES"] = str(3 * 32 * 28 * 28 * 4)  # 3 tensors per chunk -> 7 chunks
    out = subprocess.run([sys.executable, "-c", code % root], env=env, capture_output=True, text=True, timeout=300)
    assert out.returncode == 0 and "ok" in out.stdout, out.stderr[-2000:]


def test_lazy_search_mixed_batch_vs_oracle():
    """The search prices the first candidates in one pass and the rest only
    for tensors whose early-stopped scan has not stopped yet (sel_pending):
    a batch mixing shallow (sparsity 0.5: stops after 4 candidates) and deep
    (0.9+: 10 or more) searches must give every tensor the reference's N and
    container bytes."""
    sp = [0.5, 0.92, 0.5, 0.95, 0.88, 0.3]
    ts = [sz.gen_synthetic("relu-laplace", [1, 128, 28, 28], s, 700 + i) for i, s in enumerate(sp)]
    many = container.compress_many(ts, 8, format=2, block_syms=2048)
    depths = []
    for t, c in zip(ts, many):
        ref = orc.compress(t.data, t.dims, 8, None, 14, fmt=2, lanes=32, block_syms=2048)
        assert container.to_bytes(c) == orc.to_bytes(ref)
        depths.append(len(optimizer.search(t, 8)[1].candidates))
    assert min(depths) <= 5 < max(depths), depths  # both passes exercised


def test_device_header_decode_matches_host_header_path():
    """scz_decode_batch_device (headers never leave the device) reconstructs
    exactly what the host-header path does, for v1 and v2, mixed K and a
    tensor with non-finite input (its status is reported, others decode)."""
    import ctypes

    import torch

    from paper_2511_11664_b200 import _native

    dims = (1, 64, 28, 28)
    T = int(np.prod(dims))
    xs = [make_input(dict(kind="relu-laplace", dims=dims, sparsity=s, seed=90 + i))
          for i, s in enumerate([0.5, 0.9, 0.2, 0.6])]
    xs[2][17] = np.nan
    x = torch.from_numpy(np.stack(xs)).cuda()
    for fmt in (1, 2):
        ctx = _native.Context(0)
        lib = ctx.lib
        batch = _native.Batch()
        ctx.check(lib.scz_encode_batch(ctx.h, ctypes.c_void_p(x.data_ptr()), T, 4, 8, -1, 14, fmt, 32, 2048,
                                       ctypes.byref(batch)))
        out_dev = torch.full_like(x, -1.0)
        ctx.check(lib.scz_decode_batch_device(ctx.h, ctypes.c_void_p(out_dev.data_ptr())))
        st_dev = (ctypes.c_int32 * 4)()
        ctx.check(lib.scz_decode_status(ctx.h, 4, st_dev))
        info = (_native.Info * 4)()
        ctx.check(lib.scz_batch_sync(ctx.h, ctypes.byref(batch), info))
        assert [info[i].status for i in range(4)] == [0, 0, 1, 0]
        assert list(st_dev) == [0, 0, 1, 0]
        for i in (0, 1, 3):
            c = sz.compress(sz.FeatureTensor(dims, xs[i]), 8, format=fmt, block_syms=2048)
            want = sz.decompress(c).data
            assert np.array_equal(out_dev[i].cpu().numpy().view(np.uint32), want.view(np.uint32)), (fmt, i)


def test_decompress_many_mixed_versions_shapes_and_widths():
    """One batch decode over v1 and v2 containers of different shapes, K
    (the K in {1, 2, 4} row kernels, the general one, u16 symbols) and a
    tensor size that is not a multiple of 4 (unaligned output rows)."""
    specs = [
        (dict(kind="relu-laplace", dims=[1, 64, 28, 28], sparsity=0.5, seed=1), 8, None, 1),
        (dict(kind="relu-laplace", dims=[1, 64, 28, 28], sparsity=0.5, seed=2), 8, None, 2),
        (dict(kind="signed", dims=[3, 5, 7], seed=5), 6, None, 2),
        (dict(kind="relu-laplace", dims=[1, 128, 28, 28], sparsity=0.93, seed=3), 8, None, 2),
        (dict(kind="relu-laplace", dims=[1, 64, 28, 28], sparsity=0.4, seed=4), 8, 196, 2),   # K = 256: u16
        (dict(kind="relu-laplace", dims=[601], sparsity=0.3, seed=6), 5, 1, 1),
        (dict(kind="relu-laplace", dims=[1, 32, 20, 20], sparsity=0.6, seed=7), 4, 3200, 2),  # K = 4
    ]
    cs, ts = [], []
    for spec, q, n_rows, fmt in specs:
        t = sz.FeatureTensor(tuple(spec["dims"]), make_input(spec))
        ts.append(t)
        cs.append(sz.compress(t, q, n_rows, format=fmt, block_syms=1024))
    assert len({c.n_cols for c in cs}) >= 4
    outs = container.decompress_many(cs)
    for c, o in zip(cs, outs):
        want = sz.decompress(c)
        assert np.array_equal(o.data.view(np.uint32), want.data.view(np.uint32))
