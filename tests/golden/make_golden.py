"""Generate the golden vectors that pin the oracle (and through it the product).

Runs the UNMODIFIED reference package from /root/reference/pkg/src (read-only,
present only in the build container, never on the GPU box) and writes:

* ``tests/golden/golden.json`` -- manifest: per case the input spec, the
  sha256 of the input array, the reference's container bytes (sha256 + size,
  plus the file name when small enough to commit), the chosen N, the search
  report and the sha256 of ``decompress`` output bits.
* ``tests/golden/*.scz`` -- full reference containers for the small cases.
* stage-level known answers (quantize edge values, normalisation, rANS
  streams, v2 lane pins, error classes).

Usage:  python tests/golden/make_golden.py [--big]
``--big`` also runs the C4 Llama2-7B (1x2048x4096) case (~2 min of reference
CPU time).  The committed manifest was generated with --big.
"""

from __future__ import annotations

import argparse
import hashlib
import json
import os
import sys

import numpy as np

REF = "/root/reference/pkg/src"
HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, REF)
sys.path.insert(0, os.path.dirname(HERE))

from sczip import bench, container, optimizer, rans, sparse, tensor  # noqa: E402  (reference)
from sczip import errors as E  # noqa: E402

from inputs import make_input  # noqa: E402  (tests/inputs.py, our restatement)


def sha(b: bytes) -> str:
    return hashlib.sha256(b).hexdigest()


def ref_input(spec):
    """The reference's own generator for relu/uniform specs (bench.py:60-85)."""
    kind = spec["kind"]
    if kind in ("relu-laplace", "uniform", "constant"):
        return bench.gen_synthetic(kind, spec["dims"], spec.get("sparsity", 0.0), spec["seed"])
    if kind == "signed":
        t = int(np.prod(spec["dims"]))
        data = np.random.default_rng(spec["seed"]).laplace(0.0, 1.0, t).astype(np.float32)
        return tensor.FeatureTensor(tuple(spec["dims"]), data)
    raise ValueError(kind)


SMALL = [
    # reference test fixtures (test_container.py:14-16, test_optimizer.py)
    dict(kind="relu-laplace", dims=[8, 8, 8], sparsity=0.8, seed=21, q=4),
    dict(kind="relu-laplace", dims=[8, 8, 8], sparsity=0.8, seed=21, q=2),
    dict(kind="relu-laplace", dims=[8, 8, 8], sparsity=0.8, seed=21, q=8),
    dict(kind="relu-laplace", dims=[8, 8, 8], sparsity=0.8, seed=21, q=4, n_rows=64),
    dict(kind="relu-laplace", dims=[8, 9, 10], sparsity=0.85, seed=3, q=4),
    dict(kind="relu-laplace", dims=[6, 8, 10], sparsity=0.8, seed=1, q=4),
    dict(kind="relu-laplace", dims=[4, 8], sparsity=0.5, seed=0, q=4),
    dict(kind="uniform", dims=[16, 16, 4], sparsity=0.0, seed=3, q=8),
    dict(kind="uniform", dims=[4], sparsity=0.0, seed=0, q=2),
    dict(kind="constant", dims=[5, 7], seed=0, q=3),
    dict(kind="signed", dims=[3, 5, 7], seed=5, q=6),
    dict(kind="signed", dims=[64, 14, 14], seed=0, q=8),
    dict(kind="relu-laplace", dims=[600], sparsity=0.3, seed=9, q=5, n_rows=2),  # K=300 > 2^Q
    dict(kind="relu-laplace", dims=[360], sparsity=0.5, seed=4, q=3, n_rows=1),  # one row, A large
    dict(kind="relu-laplace", dims=[128, 28, 28], sparsity=0.9, seed=42, q=4),
    dict(kind="relu-laplace", dims=[1000], sparsity=0.5, seed=8, q=7, precision=8),
    dict(kind="relu-laplace", dims=[1000], sparsity=0.5, seed=8, q=7, precision=15),
    dict(kind="zeros", dims=[8, 8], q=4),
    dict(kind="zeros", dims=[16], q=4),
    dict(kind="single", dims=[1], q=4),
]

# BASELINE.json configs -- hashes only (too big to commit).
BIG = [
    dict(kind="relu-laplace", dims=[1, 512, 28, 28], sparsity=0.5, seed=42, q=8, name="C1-relu0.5"),
    dict(kind="relu-laplace", dims=[1, 512, 28, 28], sparsity=0.9, seed=42, q=8, name="C1-relu0.9"),
    dict(kind="relu-laplace", dims=[1, 256, 56, 56], sparsity=0.5, seed=0, q=8, name="C2-vgg16-s0"),
    dict(kind="signed", dims=[1, 64, 14, 14], seed=0, q=8, name="C2-mobilenetv2-s0"),
] + [
    dict(kind="signed", dims=[1, 28, 28, 192], seed=42, q=q, name=f"C5-swint-q{q}") for q in (2, 4, 6, 8)
] + [
    dict(kind="relu-laplace", dims=[1, 512, 28, 28], sparsity=0.6, seed=42, q=q,
         name=f"C5-densenet-q{q}") for q in (2, 4, 6, 8)
]
HUGE = [dict(kind="signed", dims=[1, 2048, 4096], seed=42, q=8, name="C4-llama2-7b")]


def run_case(spec, write_file):
    t = ref_input(spec) if spec["kind"] not in ("zeros", "single") else None
    if spec["kind"] == "zeros":
        t = tensor.FeatureTensor(tuple(spec["dims"]), np.zeros(int(np.prod(spec["dims"])), np.float32))
    if spec["kind"] == "single":
        t = tensor.FeatureTensor((1,), np.ones(1, np.float32))
    ours = make_input(spec)
    assert np.array_equal(ours.view(np.uint32), t.data.view(np.uint32)), spec
    q = spec["q"]
    prec = spec.get("precision", 14)
    n_rows = spec.get("n_rows")
    rec = dict(spec=spec, input_sha=sha(t.data.tobytes()))
    if n_rows is None:
        n, rep = optimizer.search(t, q)
        rec["search"] = dict(chosen=n, early_stopped=rep.early_stopped,
                             candidates=[[c.n_rows, c.n_cols, c.nnz, c.stream_len,
                                          c.entropy_bits, c.t_tot] for c in rep.candidates])
        if int(np.prod(spec["dims"])) <= 200_000:
            en, erep = optimizer.exhaustive_search(t, q)
            rec["exhaustive"] = dict(chosen=en, candidates=[[c.n_rows, c.entropy_bits, c.t_tot]
                                                            for c in erep.candidates])
    c = container.compress(t, q, n_rows, prec)
    raw = container.to_bytes(c)
    rec.update(n_rows=c.n_rows, n_cols=c.n_cols, nnz=c.nnz, scale=c.scale,
               zero_point=c.zero_point, alphabet=c.alphabet_size,
               container_sha=sha(raw), container_len=len(raw),
               payload_len=c.payload_bytes)
    out = container.decompress(c)
    rec["output_sha"] = sha(out.data.tobytes())
    if write_file:
        fname = f"case_{len(os.listdir(HERE))}_{sha(raw)[:10]}.scz"
        with open(os.path.join(HERE, fname), "wb") as f:
            f.write(raw)
        rec["file"] = fname
    # v2 lane pins: lane j of each block must equal rans.encode(block[j::W]).
    params = tensor.params_for(t, q)
    qm = tensor.quantize_reshape(t, params, c.n_rows)
    d = sparse.concat(sparse.csr_encode(qm))
    table = rans.normalize_frequencies(rans.build_counts(d, c.alphabet_size), prec)
    lanes_pin = []
    W, B = 32, 8192
    for b in range(0, min(len(d), 3 * B), B):
        blk = d.data[b:b + B]
        for j in (0, 1, 31):
            sub = blk[j::W]
            lanes_pin.append([b // B, j, sha(rans.encode(sub, table).data)])
    rec["v2_lane_pins"] = dict(lanes=W, block_syms=B, pins=lanes_pin)
    return rec


def kat_vectors():
    """Stage-level known answers taken from the reference functions."""
    out = {}
    # quantize edge values (signed/unsigned zeros, subnormals, half-way points)
    edge = np.array([0.0, -0.0, 1e-45, -1e-45, 1.17549435e-38, 3.26, 1.0, -1.0, 0.5, 2.5,
                     -2.5, 3.4e38, -3.4e38, 7.5, 6.99999, 1e-30], dtype=np.float32)
    rows = []
    for xs, q in [(edge[:12], 8), (edge, 4), (np.array([-1.0, 1.0], np.float32), 2),
                  (np.array([1e-45, 2e-45, 0.0], np.float32), 8),
                  (np.array([5.0] * 3, np.float32), 4), (np.array([-3.0] * 3, np.float32), 4)]:
        t = tensor.FeatureTensor((xs.size,), xs)
        p = tensor.params_for(t, q)
        qq, m = tensor.quantize(t, p)
        deq = tensor.dequantize(tensor.QuantizedMatrix(1, xs.size, qq, m), p, (xs.size,))
        rows.append(dict(x=xs.view(np.uint32).tolist(), q=q, scale=p.scale.hex(), z=p.zero_point,
                         sym=qq.tolist(), mask=m.tolist(), deq=deq.data.view(np.uint32).tolist()))
    out["quantize"] = rows
    # compute_params KATs (test_tensor.py:19-45)
    out["params"] = [[a, b, q, tensor.compute_params(a, b, q).scale.hex(),
                      tensor.compute_params(a, b, q).zero_point]
                     for a, b, q in [(0.0, 255.0, 8), (0.0, 7.5, 4), (-1.0, 1.0, 2), (0.0, 0.0, 4),
                                     (5.0, 5.0, 4), (-3.0, -3.0, 4), (-0.7, 3.1, 3), (-5e-40, 2e-39, 8)]]
    # normalisation on random count vectors incl. ties and starvation
    rng = np.random.default_rng(123)
    norm = []
    for i in range(60):
        a = int(rng.integers(1, 300))
        counts = rng.integers(0, 1000, a) ** int(rng.integers(1, 3))
        if i % 5 == 0:
            counts[rng.random(a) < 0.5] = 1
        if i % 7 == 0:
            counts = np.full(a, 3)
        prec = int(rng.integers(8, 16))
        try:
            f = rans.normalize_frequencies(counts, prec).freqs.tolist()
        except E.SczipError as e:
            f = type(e).__name__
        norm.append(dict(counts=counts.tolist(), precision=prec, freqs=f))
    norm.append(dict(counts=[1, 2, 3, 1, 0, 1], precision=4,
                     freqs=rans.normalize_frequencies([1, 2, 3, 1, 0, 1], 4).freqs.tolist()))
    norm.append(dict(counts=[100000, 1, 1, 1], precision=8,
                     freqs=rans.normalize_frequencies([100000, 1, 1, 1], 8).freqs.tolist()))
    out["normalize"] = norm
    # rANS streams at every precision
    streams = []
    for prec in range(8, 17):
        a = int(rng.integers(2, 200))
        n = int(rng.integers(0, 3000))
        w = rng.random(a) ** 3
        d = rng.choice(a, size=n, p=w / w.sum()).astype(np.uint32)
        if n == 0:
            d = np.zeros(1, np.uint32)
        counts = rans.build_counts(d, a)
        try:
            table = rans.normalize_frequencies(counts, prec)
        except E.SczipError:
            continue
        b = rans.encode(d, table)
        streams.append(dict(d=d.tolist(), alphabet=a, precision=prec, freqs=table.freqs.tolist(),
                            payload=b.data.hex()))
    out["rans"] = streams
    return out


def error_cases():
    """Corrupt containers and the reference's exception class for each."""
    t = bench.gen_synthetic("relu-laplace", [8, 8, 8], 0.8, 21)
    raw = container.to_bytes(container.compress(t, 4))
    cases = []

    def probe(name, blob):
        try:
            container.decompress(container.from_bytes(blob))
            cls = None
        except (E.SczipError, ValueError) as e:
            cls = type(e).__name__
        cases.append(dict(name=name, blob=blob.hex(), error=cls))

    probe("ok", raw)
    probe("bad_magic", b"NOPE" + raw[4:])
    probe("bad_version", raw[:4] + bytes([99]) + raw[5:])
    probe("truncated_payload", raw[:-3])
    probe("trailing_byte", raw + b"\x00")
    probe("short", raw[:6])
    probe("truncated_header", raw[:20])
    hdr_ab = 8 + 4 * 3 + 24 + 16
    probe("alphabet_inflated", raw[:hdr_ab] + (10**6).to_bytes(4, "little") + raw[hdr_ab + 4:])
    flip = bytearray(raw)
    flip[-5] ^= 0xFF
    probe("payload_bitflip", bytes(flip))
    flip = bytearray(raw)
    flip[8 + 12 + 8] ^= 0x01  # N field
    probe("geometry", bytes(flip))
    flip = bytearray(raw)
    flip[5] = 9  # q_bits 9 -> QuantParams InvalidInput after a clean decode
    probe("bad_qbits", bytes(flip))
    return cases


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--big", action="store_true")
    args = ap.parse_args()
    for f in os.listdir(HERE):
        if f.endswith(".scz"):
            os.unlink(os.path.join(HERE, f))
    manifest = dict(reference="/root/reference/pkg/src/sczip (unmodified)",
                    numpy=np.__version__, small=[], big=[])
    for spec in SMALL:
        manifest["small"].append(run_case(spec, write_file=True))
        print("small", spec, manifest["small"][-1]["n_rows"], flush=True)
    for spec in BIG + (HUGE if args.big else []):
        manifest["big"].append(run_case(spec, write_file=False))
        print("big", spec["name"], manifest["big"][-1]["n_rows"], flush=True)
    manifest["kat"] = kat_vectors()
    manifest["errors"] = error_cases()
    with open(os.path.join(HERE, "golden.json"), "w") as f:
        json.dump(manifest, f, indent=1)
    print("wrote", os.path.join(HERE, "golden.json"))


if __name__ == "__main__":
    main()
