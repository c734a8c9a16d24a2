"""Host-side harness rows of SURVEY.md 8(f): the channel model (pinned to
values computed with the unmodified reference, channel.py:58-68) and the
measure / run_sweep CSV harness (bench.py:101-186) over the GPU path."""

import csv
import math

import numpy as np
import pytest

import paper_2511_11664_b200 as sz
from paper_2511_11664_b200 import bench, channel
from paper_2511_11664_b200.errors import InvalidInput


def test_channel_matches_reference_values():
    # sczip.channel with default params / from_db(20e6, 3.0, 0.5, 0.01), run in this container
    p = channel.ChannelParams()
    assert channel.outage_rate(p) == 143624.39778969807
    assert channel.comm_latency(8 * 266247, p) == 14.830182286430304
    q = channel.ChannelParams.from_db(20e6, 3.0, 0.5, 0.01)
    assert channel.outage_rate(q) == 287863.71273872047
    assert channel.comm_latency(123456, q) == 0.4288696161994369


@pytest.mark.parametrize("kw", [dict(bandwidth_hz=0), dict(mean_snr=-1.0), dict(fading_var=0.0),
                                dict(outage_prob=1.0), dict(outage_prob=0.0)])
def test_channel_rejects_bad_params(kw):
    with pytest.raises(InvalidInput):
        channel.ChannelParams(**kw)
    with pytest.raises(InvalidInput):
        channel.comm_latency(-1, channel.ChannelParams())


def test_csv_schema_is_the_reference_one(tmp_path):
    rec = bench.BenchRecord("t", 8, 4, 2, 3, 1.5, 60, 10, 70, 0.1, 0.0, 0.2, 0.0, 1e-4, 0.01)
    path = tmp_path / "r.csv"
    bench.write_csv([rec], path)
    rows = list(csv.reader(open(path)))
    assert rows[0] == bench.CSV_COLUMNS
    assert rows[1][0] == "t" and rows[1][1] == "8" and len(rows[1]) == len(bench.CSV_COLUMNS)


@pytest.mark.gpu
def test_measure_and_sweep_on_gpu(tmp_path):
    t = sz.gen_synthetic("relu-laplace", [1, 32, 28, 28], 0.5, 3)
    path = tmp_path / "sweep.csv"
    recs = bench.run_sweep(t, [4, 8], repetitions=3, csv_path=path)
    assert [r.Q for r in recs] == [4, 8]
    for r in recs:
        c = sz.compress(t, r.Q, r.N)
        assert (r.N, r.K, r.nnz, r.total_bytes) == (c.n_rows, c.n_cols, c.nnz, c.total_bytes)
        assert r.max_abs_err <= c.scale * (1 + 1e-6)
        assert math.isclose(r.t_comm_s, channel.comm_latency(8 * c.payload_bytes, channel.ChannelParams()))
        assert r.enc_ms > 0 and r.dec_ms > 0
    rows = list(csv.reader(open(path)))
    assert rows[0] == bench.CSV_COLUMNS and len(rows) == 3
    # explicit reshapes: an infeasible one is skipped row-wise, not fatal
    recs = bench.run_sweep(t, [8], n_policy=[25088, 5], repetitions=2)
    assert [r.N for r in recs] == [25088]
    # v2 containers through the same harness
    r2 = bench.measure(t, 8, None, repetitions=2, format=2, block_syms=1024)
    assert r2.total_bytes > 0 and np.isfinite(r2.entropy_bits)
