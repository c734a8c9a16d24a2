"""Byte-level parity of the exact device path bench.py times, and of the
general-alphabet classes, against the CPU oracle.

bench.py's step is scz_encode_batch -> scz_batch_sync ->
scz_decode_batch_async over a device-resident batch (and, for the latency /
device-header variants, scz_decode_batch_device).  These tests run that call
sequence on seeded batches of the BASELINE configs (VGG16 and MobileNetV2
split features, v2 with 8192-symbol blocks and v1), rebuild every container
from the device buffers, and compare it byte for byte with
oracle.compress (the reference's algorithm; container.py:73-134) and every
reconstruction bit for bit with oracle.decompress (container.py:109-121).

The general-alphabet cases push K past 65535 (u32 symbols), the alphabet
past 8192 (encoder tables in global memory) and past 4096 (the decoder's
binary-search class) through the container API, in both formats.
"""

import ctypes
import ctypes.util

import numpy as np
import pytest

import paper_2511_11664_b200 as sz
from oracle import oracle as orc
from paper_2511_11664_b200 import _native, container
from inputs import GENERAL_ALPHABET, make_input, sparse_columns

pytestmark = pytest.mark.gpu

_cudart = None


def cudart():
    global _cudart
    if _cudart is None:
        import glob

        cands = glob.glob("/usr/local/cuda/lib64/libcudart.so*") + [ctypes.util.find_library("cudart") or ""]
        for c in cands:
            if c:
                try:
                    _cudart = ctypes.CDLL(c)
                    break
                except OSError:
                    continue
        assert _cudart is not None, "libcudart not found"
        _cudart.cudaMemcpy.argtypes = [ctypes.c_void_p, ctypes.c_void_p, ctypes.c_size_t, ctypes.c_int]
    return _cudart


def d2h(ptr: int, nbytes: int) -> np.ndarray:
    out = np.empty(max(nbytes, 1), np.uint8)
    if nbytes:
        assert cudart().cudaMemcpy(out.ctypes.data, ctypes.c_void_p(ptr), nbytes, 2) == 0
    return out[:nbytes]


def device_batch_containers(ctx, batch, infos, B, dims):
    """Containers of a synced scz_batch, read straight from its device buffers."""
    pay = d2h(batch.d_payload, int(batch.payload_total))
    fr = d2h(batch.d_freqs, 4 * int(batch.freqs_total)).view(np.uint32)
    bl = d2h(batch.d_block_bytes, 4 * int(batch.blocks_total)).view(np.uint32)
    out = []
    for i in range(B):
        inf = infos[i]
        assert inf.status == 0, (i, inf.status)
        freqs = fr[inf.freqs_off: inf.freqs_off + inf.alphabet].astype(np.int64)
        blocks = bl[inf.blocks_off: inf.blocks_off + inf.n_blocks].copy() if inf.version == 2 else None
        payload = pay[inf.payload_off: inf.payload_off + inf.payload_len].tobytes()
        out.append(container._container_from_info(inf, dims, freqs, blocks, payload))
    return out


WORKLOADS = [
    # (name, dims, kind, sparsity, batch) -- BASELINE configs[1] at bench settings
    ("vgg16", (1, 256, 56, 56), "relu-laplace", 0.5, 16),
    ("mobilenetv2", (1, 64, 14, 14), "signed", 0.0, 256),
]


@pytest.mark.parametrize("fmt", [2, 1])
@pytest.mark.parametrize("wl", WORKLOADS, ids=[w[0] for w in WORKLOADS])
def test_bench_device_path_bit_exact(wl, fmt):
    import torch

    name, dims, kind, sparsity, B = wl
    T = int(np.prod(dims))
    xs = np.stack([make_input(dict(kind=kind, dims=dims, sparsity=sparsity, seed=s)) for s in range(B)])
    x = torch.from_numpy(xs).cuda()
    out = torch.full_like(x, -7.0)
    ctx = _native.Context(0)
    lib = ctx.lib
    batch = _native.Batch()
    infos = (_native.Info * B)()
    bs = 8192
    for rep in range(3):  # eager, graph capture, graph replay: all three must be exact
        out.fill_(-7.0)
        ctx.check(lib.scz_encode_batch(ctx.h, ctypes.c_void_p(x.data_ptr()), T, B, 8, -1, 14, fmt, 32, bs,
                                       ctypes.byref(batch)))
        ctx.check(lib.scz_batch_sync(ctx.h, ctypes.byref(batch), infos))
        ctx.check(lib.scz_decode_batch_async(ctx.h, infos, B, ctypes.c_void_p(batch.d_freqs),
                                             ctypes.c_void_p(batch.d_block_bytes), ctypes.c_void_p(batch.d_payload),
                                             ctypes.c_void_p(out.data_ptr())))
        st = (ctypes.c_int32 * B)()
        ctx.check(lib.scz_decode_status(ctx.h, B, st))
        assert list(st) == [0] * B
        if rep == 0:
            got = device_batch_containers(ctx, batch, infos, B, dims)
            refs = [orc.compress(xs[i], dims, 8, None, 14, fmt=fmt, lanes=32, block_syms=bs) for i in range(B)]
            for i in range(B):
                assert container.to_bytes(got[i]) == orc.to_bytes(refs[i]), (name, fmt, i)
            want = np.stack([orc.decompress(r) for r in refs])
        assert np.array_equal(out.cpu().numpy().view(np.uint32), want.view(np.uint32)), (name, fmt, rep)
    # the device-header decode of the same encode (no host round trip)
    out.fill_(-7.0)
    ctx.check(lib.scz_decode_batch_device(ctx.h, ctypes.c_void_p(out.data_ptr())))
    st = (ctypes.c_int32 * B)()
    ctx.check(lib.scz_decode_status(ctx.h, B, st))
    assert list(st) == [0] * B
    assert np.array_equal(out.cpu().numpy().view(np.uint32), want.view(np.uint32)), (name, fmt, "device headers")


@pytest.mark.parametrize("fmt", [2, 1])
def test_unaligned_device_inputs(fmt):
    """Tensors whose fp32 data starts off a 16-byte boundary (an odd element
    count and a one-element offset into the allocation): the statistics and
    quantiser kernels take their bounds-checked scalar loads, and the
    containers and reconstructions still equal the oracle's.  The decode
    output goes to an unaligned destination too."""
    import torch

    B, T, q = 4, 40001, 8
    xs = np.stack([make_input(dict(kind="relu-laplace", dims=(T,), sparsity=0.5, seed=100 + s)) for s in range(B)])
    buf = torch.zeros(B * T + 3, dtype=torch.float32, device="cuda")
    x = buf[1: 1 + B * T]
    x.copy_(torch.from_numpy(xs.ravel()))
    obuf = torch.full((B * T + 3,), -7.0, dtype=torch.float32, device="cuda")
    out = obuf[3: 3 + B * T]
    ctx = _native.Context(0)
    lib = ctx.lib
    batch = _native.Batch()
    infos = (_native.Info * B)()
    ctx.check(lib.scz_encode_batch(ctx.h, ctypes.c_void_p(x.data_ptr()), T, B, q, -1, 14, fmt, 32, 2048,
                                   ctypes.byref(batch)))
    ctx.check(lib.scz_batch_sync(ctx.h, ctypes.byref(batch), infos))
    ctx.check(lib.scz_decode_batch_async(ctx.h, infos, B, ctypes.c_void_p(batch.d_freqs),
                                         ctypes.c_void_p(batch.d_block_bytes), ctypes.c_void_p(batch.d_payload),
                                         ctypes.c_void_p(out.data_ptr())))
    st = (ctypes.c_int32 * B)()
    ctx.check(lib.scz_decode_status(ctx.h, B, st))
    assert list(st) == [0] * B
    got = device_batch_containers(ctx, batch, infos, B, (T,))
    refs = [orc.compress(xs[i], (T,), q, None, 14, fmt=fmt, lanes=32, block_syms=2048) for i in range(B)]
    for i in range(B):
        assert container.to_bytes(got[i]) == orc.to_bytes(refs[i]), (fmt, i)
    want = np.stack([orc.decompress(r) for r in refs]).ravel()
    assert np.array_equal(out.cpu().numpy().view(np.uint32), want.view(np.uint32)), fmt


GENERAL = GENERAL_ALPHABET


@pytest.mark.parametrize("case", GENERAL, ids=[g[0] for g in GENERAL])
@pytest.mark.parametrize("fmt", [1, 2])
def test_general_alphabet_containers_vs_oracle(case, fmt):
    label, T, n_rows, stride, q, prec = case
    x = sparse_columns(T, T // n_rows, stride, seed=T % 997)
    t = sz.FeatureTensor((T,), x)
    ref = orc.compress(x, (T,), q, n_rows, prec, fmt=fmt, lanes=32, block_syms=4096)
    assert len(ref["freqs"]) > 256, label
    c = sz.compress(t, q, n_rows, prec, format=fmt, block_syms=4096)
    assert container.to_bytes(c) == orc.to_bytes(ref), (label, fmt)
    out = sz.decompress(container.from_bytes(container.to_bytes(c)))
    assert np.array_equal(out.data.view(np.uint32), orc.decompress(ref).view(np.uint32)), (label, fmt)
    # batch path (scz_compress_batch / scz_decompress_batch) over the same class
    many = container.compress_many([t, t], q, n_rows, prec, format=fmt, block_syms=4096)
    assert all(container.to_bytes(m) == orc.to_bytes(ref) for m in many)
    outs = container.decompress_many(many)
    assert all(np.array_equal(o.data, out.data) for o in outs)


def test_general_alphabet_precision_too_small():
    """More distinct symbols than 2^precision slots: PrecisionTooSmall, as the reference."""
    from paper_2511_11664_b200.errors import PrecisionTooSmall

    T, n_rows = 40000 * 5, 5
    x = sparse_columns(T, T // n_rows, 1, seed=3)  # ~40000 distinct column symbols > 2^14
    with pytest.raises(orc.OracleError):
        orc.compress(x, (T,), 8, n_rows, 14)
    with pytest.raises(PrecisionTooSmall):
        sz.compress(sz.FeatureTensor((T,), x), 8, n_rows, 14)


def test_back_to_back_async_decodes_on_one_context():
    """Two scz_decode_batch_async calls queued on one context behind a long
    encode, without a host sync between them: each must decode its own
    headers (the pinned header staging rotates)."""
    import torch

    dims_a, dims_b = (1, 64, 28, 28), (1, 32, 14, 14)
    Ta, Tb = int(np.prod(dims_a)), int(np.prod(dims_b))
    xa = np.stack([make_input(dict(kind="relu-laplace", dims=dims_a, sparsity=0.5, seed=40 + i)) for i in range(4)])
    xb = np.stack([make_input(dict(kind="signed", dims=dims_b, seed=60 + i)) for i in range(3)])
    big = torch.from_numpy(np.stack([make_input(dict(kind="relu-laplace", dims=(1, 256, 56, 56), sparsity=0.5,
                                                     seed=i)) for i in range(32)])).cuda()
    ca, cb, cd = _native.Context(0), _native.Context(0), _native.Context(0)
    lib = ca.lib
    da, db = torch.from_numpy(xa).cuda(), torch.from_numpy(xb).cuda()
    ba, bb, bbig = _native.Batch(), _native.Batch(), _native.Batch()
    ia, ib = (_native.Info * 4)(), (_native.Info * 3)()
    ca.check(lib.scz_encode_batch(ca.h, ctypes.c_void_p(da.data_ptr()), Ta, 4, 8, -1, 14, 2, 32, 2048, ctypes.byref(ba)))
    ca.check(lib.scz_batch_sync(ca.h, ctypes.byref(ba), ia))
    cb.check(lib.scz_encode_batch(cb.h, ctypes.c_void_p(db.data_ptr()), Tb, 3, 6, -1, 14, 2, 32, 1024, ctypes.byref(bb)))
    cb.check(lib.scz_batch_sync(cb.h, ctypes.byref(bb), ib))
    want_a = [sz.decompress(sz.compress(sz.FeatureTensor(dims_a, x), 8, format=2, block_syms=2048)).data for x in xa]
    want_b = [sz.decompress(sz.compress(sz.FeatureTensor(dims_b, x), 6, format=2, block_syms=1024)).data for x in xb]
    for _ in range(3):
        oa, ob = torch.full_like(da, -1.0), torch.full_like(db, -1.0)
        torch.cuda.synchronize()
        # a long encode on the decoder's context delays both queued header copies
        cd.check(lib.scz_encode_batch(cd.h, ctypes.c_void_p(big.data_ptr()), big.shape[1], 32, 8, -1, 14, 2, 32,
                                      8192, ctypes.byref(bbig)))
        cd.check(lib.scz_decode_batch_async(cd.h, ia, 4, ctypes.c_void_p(ba.d_freqs), ctypes.c_void_p(ba.d_block_bytes),
                                            ctypes.c_void_p(ba.d_payload), ctypes.c_void_p(oa.data_ptr())))
        cd.check(lib.scz_decode_batch_async(cd.h, ib, 3, ctypes.c_void_p(bb.d_freqs), ctypes.c_void_p(bb.d_block_bytes),
                                            ctypes.c_void_p(bb.d_payload), ctypes.c_void_p(ob.data_ptr())))
        st = (ctypes.c_int32 * 3)()
        cd.check(lib.scz_decode_status(cd.h, 3, st))
        torch.cuda.synchronize()
        assert list(st) == [0, 0, 0]
        for i in range(4):
            assert np.array_equal(oa[i].cpu().numpy().view(np.uint32), want_a[i].view(np.uint32)), i
        for i in range(3):
            assert np.array_equal(ob[i].cpu().numpy().view(np.uint32), want_b[i].view(np.uint32)), i


def test_device_header_decode_refuses_a_stale_batch():
    """scz_decode_batch_device after another encode on the context (which
    reuses the encode buffers) fails cleanly instead of decoding stale data."""
    import torch

    from paper_2511_11664_b200.errors import InvalidInput

    dims = (1, 32, 28, 28)
    T = int(np.prod(dims))
    x = torch.from_numpy(np.stack([make_input(dict(kind="relu-laplace", dims=dims, sparsity=0.5, seed=i))
                                   for i in range(2)])).cuda()
    ctx = _native.Context(0)
    b = _native.Batch()
    ctx.check(ctx.lib.scz_encode_batch(ctx.h, ctypes.c_void_p(x.data_ptr()), T, 2, 8, -1, 14, 2, 32, 2048,
                                       ctypes.byref(b)))
    out = torch.empty_like(x)
    ctx.check(ctx.lib.scz_decode_batch_device(ctx.h, ctypes.c_void_p(out.data_ptr())))
    # a host-buffer compress on the same context overwrites the batch buffers
    info = _native.Info()
    fp, bp, pp = (ctypes.POINTER(ctypes.c_uint32)(), ctypes.POINTER(ctypes.c_uint32)(),
                  ctypes.POINTER(ctypes.c_uint8)())
    xs = x[0].cpu().numpy()
    ctx.check(ctx.lib.scz_compress(ctx.h, _native.ptr(xs), T, 8, -1, 14, 2, 32, 2048, ctypes.byref(info),
                                   ctypes.byref(fp), ctypes.byref(bp), ctypes.byref(pp)))
    with pytest.raises(InvalidInput):
        ctx.check(ctx.lib.scz_decode_batch_device(ctx.h, ctypes.c_void_p(out.data_ptr())))


def test_highly_composite_element_count_searches_all_candidates():
    """T = 3,326,400 has 82 feasible reshapes at Q = 8 (more than
    the 64 a launch used to price): Algorithm 1 on the device picks the
    reference's N and the containers match the oracle."""
    T = 3_326_400
    assert len(orc.candidate_rows(T, 8)) > 64
    for sp, seed in ((0.5, 1), (0.95, 2)):
        x = make_input(dict(kind="relu-laplace", dims=(1, 60, 55440), sparsity=sp, seed=seed))
        t = sz.FeatureTensor((1, 60, 55440), x)
        ref = orc.compress(x, t.dims, 8, None, 14, fmt=2, lanes=32, block_syms=8192)
        c = sz.compress(t, 8, format=2)
        assert container.to_bytes(c) == orc.to_bytes(ref), sp
        n_dev, rep = sz.optimizer.exhaustive_search(t, 8)
        n_ref, seen = orc.exhaustive_search(x, 8)
        assert n_dev == n_ref and len(rep.candidates) == len(seen) > 64


@pytest.mark.parametrize("fmt", [1, 2])
def test_mixed_symbol_classes_in_one_batch_decode(fmt):
    """One batch decode whose tensors decode into different symbol classes
    (u16 rows for K = 256, u8 rows for K = 4): every tensor's row of decoded
    symbols has its own byte range (a u16 row used to overlap the u8 rows of
    later tensors when rows were indexed in elements of each class)."""
    dims = (1, 64, 28, 28)
    T = int(np.prod(dims))
    ts = [sz.FeatureTensor(dims, make_input(dict(kind="relu-laplace", dims=dims, sparsity=0.5, seed=300 + i)))
          for i in range(6)]
    cs = []
    for i, t in enumerate(ts):
        n_rows = T // 256 if i in (0, 1) else T // 4  # K = 256 -> u16 symbols; K = 4 -> u8
        cs.append(sz.compress(t, 8, n_rows, format=fmt, block_syms=1024))
    assert cs[0].n_cols == 256 and cs[2].n_cols == 4
    outs = container.decompress_many(cs)
    for c, o in zip(cs, outs):
        want = sz.decompress(c)
        assert np.array_equal(o.data.view(np.uint32), want.data.view(np.uint32))


@pytest.mark.parametrize("fmt", [2, 1])
def test_heterogeneous_device_batch_encode(fmt):
    """scz_encode_batch_ptrs: tensors of several sizes at
    arbitrary device addresses, interleaved, one of them non-finite; every
    container equals the oracle's, the failed tensor reports InvalidInput, and
    one batch decode reconstructs the rest in the caller's order."""
    import torch

    shapes = [(1, 64, 28, 28), (3, 5, 7), (1, 32, 14, 14), (1, 64, 28, 28), (601,), (1, 32, 14, 14),
              (1, 64, 28, 28)]
    specs = [dict(kind="relu-laplace" if i % 2 == 0 else "signed", dims=d, sparsity=0.5, seed=400 + i)
             for i, d in enumerate(shapes)]
    xs = [make_input(sp).astype(np.float32) for sp in specs]
    xs[5][7] = np.inf
    # tensors 0 and 3 share one [2][T] device array in order (a group used in place
    # needs consecutive addresses; here they are not consecutive in the batch, so the
    # group {0, 3, 6} is gathered), the others are separate allocations
    pair = torch.from_numpy(np.stack([xs[0], xs[3]])).cuda()
    dev = [pair[0], torch.from_numpy(xs[1]).cuda(), torch.from_numpy(xs[2]).cuda(), pair[1],
           torch.from_numpy(xs[4]).cuda(), torch.from_numpy(xs[5]).cuda(), torch.from_numpy(xs[6]).cuda()]
    B = len(dev)
    ptrs = (ctypes.c_void_p * B)(*[t.data_ptr() for t in dev])
    numel = (ctypes.c_uint64 * B)(*[t.numel() for t in dev])
    ctx = _native.Context(0)
    lib = ctx.lib
    batch = _native.Batch()
    infos = (_native.Info * B)()
    for rep in range(2):
        ctx.check(lib.scz_encode_batch_ptrs(ctx.h, ptrs, numel, B, 8, -1, 14, fmt, 32, 1024, ctypes.byref(batch)))
        ctx.check(lib.scz_batch_sync(ctx.h, ctypes.byref(batch), infos))
        assert [infos[i].status for i in range(B)] == [0, 0, 0, 0, 0, 1, 0]
        ok = [i for i in range(B) if infos[i].status == 0]
        pay = d2h(batch.d_payload, int(batch.payload_total))
        fr = d2h(batch.d_freqs, 4 * int(batch.freqs_total)).view(np.uint32)
        bl = d2h(batch.d_block_bytes, 4 * int(batch.blocks_total)).view(np.uint32)
        for i in ok:
            inf = infos[i]
            freqs = fr[inf.freqs_off: inf.freqs_off + inf.alphabet].astype(np.int64)
            blocks = bl[inf.blocks_off: inf.blocks_off + inf.n_blocks].copy() if fmt == 2 else None
            c = container._container_from_info(inf, shapes[i], freqs, blocks,
                                               pay[inf.payload_off: inf.payload_off + inf.payload_len].tobytes())
            ref = orc.compress(xs[i], shapes[i], 8, None, 14, fmt=fmt, lanes=32, block_syms=1024)
            assert container.to_bytes(c) == orc.to_bytes(ref), (i, rep)
        # one batch decode of the good tensors (their infos index the combined buffers)
        sub = (_native.Info * len(ok))(*[infos[i] for i in ok])
        tot = sum(dev[i].numel() for i in ok)
        out = torch.full((tot,), -1.0, device="cuda")
        ctx.check(lib.scz_decode_batch_async(ctx.h, sub, len(ok), ctypes.c_void_p(batch.d_freqs),
                                             ctypes.c_void_p(batch.d_block_bytes), ctypes.c_void_p(batch.d_payload),
                                             ctypes.c_void_p(out.data_ptr())))
        st = (ctypes.c_int32 * len(ok))()
        ctx.check(lib.scz_decode_status(ctx.h, len(ok), st))
        assert list(st) == [0] * len(ok)
        got = out.cpu().numpy()
        pos = 0
        for i in ok:
            want = orc.decompress(orc.compress(xs[i], shapes[i], 8, None, 14, fmt=fmt, lanes=32, block_syms=1024))
            assert np.array_equal(got[pos: pos + xs[i].size].view(np.uint32), want.view(np.uint32)), (i, rep)
            pos += xs[i].size


def test_compress_many_mixed_shapes():
    """container.compress_many groups mixed shapes and keeps the input order."""
    shapes = [(1, 32, 14, 14), (3, 5, 7), (1, 32, 14, 14), (601,)]
    ts = [sz.FeatureTensor(d, make_input(dict(kind="relu-laplace", dims=d, sparsity=0.4, seed=i)))
          for i, d in enumerate(shapes)]
    for fmt in (1, 2):
        many = container.compress_many(ts, 6, format=fmt, block_syms=512)
        for t, c in zip(ts, many):
            assert c.dims == t.dims
            assert container.to_bytes(c) == container.to_bytes(sz.compress(t, 6, format=fmt, block_syms=512))
        outs = container.decompress_many(many)
        for c, o in zip(many, outs):
            assert np.array_equal(o.data.view(np.uint32), sz.decompress(c).data.view(np.uint32))
