"""File and wire I/O either side of the path and the GPU-routed CLI
(SURVEY.md 8f rows 1 and 3): RTF tensors (tensor.py:183-208), container
files (container.py:183-190), optimizer.write_report_csv
(optimizer.py:169-184) and the sczip command line (cli.py:1-150).
CPU tests cover the host code; -m gpu tests drive the CLI end to end."""

import csv
import os

import numpy as np
import pytest

import paper_2511_11664_b200 as sz
from paper_2511_11664_b200 import cli, container, optimizer, tensor
from paper_2511_11664_b200.errors import InvalidInput, UnsupportedVersion

GOLDEN = os.path.join(os.path.dirname(__file__), "golden")


def test_rtf_round_trip_and_layout(tmp_path):
    x = np.array([0.0, -1.5, 3.25, np.float32(1e-30), -0.0, 7.0], np.float32)
    t = sz.FeatureTensor((2, 3), x)
    p = tmp_path / "t.rtf"
    tensor.write_rtf(t, p)
    raw = p.read_bytes()
    # "RTF1" | u8 rank | u32 dims | f32 data, little-endian
    assert raw[:4] == b"RTF1" and raw[4] == 2
    assert np.frombuffer(raw[5:13], "<u4").tolist() == [2, 3] and len(raw) == 13 + 4 * 6
    back = tensor.read_rtf(p)
    assert back.dims == (2, 3) and np.array_equal(back.data.view(np.uint32), x.view(np.uint32))


@pytest.mark.parametrize("blob", [b"", b"RTF", b"XXXX\x01\x00\x00\x00\x01", b"RTF1\x02\x01\x00\x00\x00",
                                  b"RTF1\x01\x02\x00\x00\x00" + b"\0" * 4])
def test_rtf_malformed_files_raise_invalid_input(tmp_path, blob):
    p = tmp_path / "bad.rtf"
    p.write_bytes(blob)
    with pytest.raises(InvalidInput):
        tensor.read_rtf(p)


def test_rtf_rejects_non_finite_payload(tmp_path):
    p = tmp_path / "nan.rtf"
    p.write_bytes(b"RTF1\x01\x02\x00\x00\x00" + np.array([1.0, np.nan], "<f4").tobytes())
    with pytest.raises(InvalidInput):
        tensor.read_rtf(p)


def test_container_files_round_trip_v1_golden_and_v2(golden, tmp_path):
    for rec in golden["small"][:6]:
        raw = open(os.path.join(GOLDEN, rec["file"]), "rb").read()
        c = container.from_bytes(raw)
        p = tmp_path / rec["file"]
        container.write_container(c, p)
        assert p.read_bytes() == raw
        c2 = container.read_container(p)
        assert container.to_bytes(c2) == raw and c2.header_bytes + c2.payload_bytes == len(raw)
    # a v2 container (FORMAT.md) written and read back; the reference parser
    # rule (version byte) makes it UnsupportedVersion for a v1-only reader
    v1 = container.from_bytes(open(os.path.join(GOLDEN, golden["small"][0]["file"]), "rb").read())
    v2 = container.Container(v1.q_bits, v1.precision, v1.dims, v1.n_rows, v1.n_cols, v1.nnz, v1.scale,
                             v1.zero_point, v1.freqs, v1.payload, version=2, lanes=32, block_syms=256,
                             block_bytes=np.array([len(v1.payload)], np.uint32))
    p = tmp_path / "v2.scz"
    container.write_container(v2, p)
    back = container.read_container(p)
    assert back.version == 2 and back.block_syms == 256 and list(back.block_bytes) == [len(v1.payload)]
    assert container.to_bytes(back) == p.read_bytes()
    bad = bytearray(p.read_bytes())
    bad[4] = 9
    with pytest.raises(UnsupportedVersion):
        container.from_bytes(bytes(bad))


def test_write_report_csv_schema(tmp_path):
    rep = optimizer.SearchReport()
    rep.candidates = [optimizer.CostBreakdown(100352, 4, 200684, 501720, 4.1234567, 2068800.1234),
                      optimizer.CostBreakdown(50176, 8, 200684, 451544, 4.6, 2077102.4)]
    rep.chosen = 100352
    p = tmp_path / "r.csv"
    optimizer.write_report_csv(rep, p)
    rows = list(csv.reader(open(p)))
    assert rows[0] == ["N", "K", "nnz", "entropy_bits_per_symbol", "t_tot_bits", "chosen"]
    assert rows[1] == ["100352", "4", "200684", "4.123457", "2068800.123", "1"]
    assert rows[2][-1] == "0" and len(rows) == 3


@pytest.mark.parametrize("argv", [[], ["compress", "--bogus"], ["compress", "x.rtf", "-o", "y.scz"],
                                  ["nosuch"], ["analyze", "x.rtf"]])
def test_cli_usage_errors_exit_1(argv, capsys):
    assert cli.cli_dispatch(argv) == 1


def test_cli_data_errors_exit_2(tmp_path, capsys):
    bad = tmp_path / "bad.rtf"
    bad.write_bytes(b"garbage")
    assert cli.cli_dispatch(["compress", str(bad), "--q", "4", "-o", str(tmp_path / "o.scz")]) == 2
    assert cli.cli_dispatch(["latency", str(tmp_path / "missing.scz")]) == 2


def test_cli_latency_env_and_flags(golden, tmp_path, capsys, monkeypatch):
    path = os.path.join(GOLDEN, golden["small"][0]["file"])
    c = container.read_container(path)
    monkeypatch.setenv("SCZ_BW_HZ", "20e6")
    assert cli.cli_dispatch(["latency", path]) == 0
    out = capsys.readouterr().out
    link = sz.ChannelParams.from_db(bandwidth_hz=20e6)
    assert f"payload_bits={8 * c.payload_bytes}" in out
    assert f"t_comm_s={sz.comm_latency(8 * c.payload_bytes, link):.9g}" in out
    assert cli.cli_dispatch(["latency", path, "--bw-hz", "5e6"]) == 0
    assert f"rate_bps={sz.outage_rate(sz.ChannelParams.from_db(bandwidth_hz=5e6)):.1f}" in capsys.readouterr().out


@pytest.mark.gpu
@pytest.mark.parametrize("fmt", [1, 2])
def test_cli_compress_decompress_analyze_on_gpu(tmp_path, capsys, fmt):
    from oracle import oracle as orc

    t = sz.gen_synthetic("relu-laplace", [1, 64, 28, 28], 0.6, 5)
    src = tmp_path / "in.rtf"
    tensor.write_rtf(t, src)
    scz, back, rep = tmp_path / "o.scz", tmp_path / "back.rtf", tmp_path / "rep.csv"
    assert cli.cli_dispatch(["compress", str(src), "--q", "8", "-o", str(scz), "--format", str(fmt),
                             "--block-syms", "2048"]) == 0
    ref = orc.compress(t.data, t.dims, 8, None, 14, fmt=fmt, lanes=32, block_syms=2048)
    assert scz.read_bytes() == orc.to_bytes(ref)
    assert cli.cli_dispatch(["decompress", str(scz), "-o", str(back)]) == 0
    out = tensor.read_rtf(back)
    assert np.array_equal(out.data.view(np.uint32), orc.decompress(ref).view(np.uint32))
    assert cli.cli_dispatch(["analyze", str(src), "--q", "8", "--csv", str(rep)]) == 0
    n_ex, seen = orc.exhaustive_search(t.data, 8)
    rows = list(csv.reader(open(rep)))[1:]
    assert [int(r[0]) for r in rows] == [int(c[0]) for c in seen]
    assert [r[0] for r in rows if r[-1] == "1"] == [str(n_ex)]
    printed = capsys.readouterr().out
    assert "chosen" in printed and "*" in printed


@pytest.mark.gpu
def test_measure_times_are_cuda_events(tmp_path):
    """bench.measure's enc_ms / dec_ms come from scz_last_call_ms (CUDA events
    around the call's copies and kernels): positive, and below the wall time
    of the same Python call."""
    import time

    from paper_2511_11664_b200 import _native, bench

    t = sz.gen_synthetic("relu-laplace", [1, 64, 56, 56], 0.5, 1)
    r = bench.measure(t, 8, None, repetitions=5)
    t0 = time.perf_counter()
    sz.compress(t, 8, r.N)
    wall = (time.perf_counter() - t0) * 1e3
    dev = _native.context().last_call_ms()
    assert 0 < dev <= wall and 0 < r.enc_ms and 0 < r.dec_ms
