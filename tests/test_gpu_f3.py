"""f3: the raw collection outside HBM, through the C ABI vs the oracle.

* paris_summarize over HOST raw (pageable and pinned): the double-buffered chunked
  H2D pipeline (the Coordinator / IndexBulkLoading double buffer, PAPER.md
  P:459-465) must give the same SAX array as the device-resident path and match the
  oracle; many chunks (forced small through PARIS_HOST_CHUNK_BYTES) with a ragged
  last chunk and every kernel variant (TMA-tiled, fast, generic).
* paris_knn_exact / paris_knn_index / paris_knn_nb with raw in PINNED host memory
  (only the candidates' rows are read, through the mapping): exact results equal to
  the device-raw run and to the oracle; pageable raw is rejected (PARIS_EINVAL).
"""
import ctypes
import os

import numpy as np
import pytest

import datagen
import oracle
from tests._parity import check_knn, sax_mismatches

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def P():
    import __graft_entry__ as ge
    ge.build()
    import paper_2009_00166_b200 as p
    return p


@pytest.fixture()
def small_chunks():
    old = os.environ.get("PARIS_HOST_CHUNK_BYTES")
    os.environ["PARIS_HOST_CHUNK_BYTES"] = str(1 << 20)  # 1 MB: 1024 series of 256 per chunk
    yield
    if old is None:
        del os.environ["PARIS_HOST_CHUNK_BYTES"]
    else:
        os.environ["PARIS_HOST_CHUNK_BYTES"] = old


@pytest.mark.parametrize("pinned", [False, True])
@pytest.mark.parametrize("n,length,w,card", [(20_000, 256, 16, 256), (20_003, 256, 16, 256),
                                             (9_001, 128, 8, 64), (5_000, 100, 5, 16),
                                             (1, 256, 16, 256), (15, 512, 16, 256)])
def test_summarize_host_raw(P, small_chunks, pinned, n, length, w, card):
    import torch
    x = datagen.random_walks(n, length, 31 + n + length)
    h = torch.from_numpy(x)
    if pinned:
        h = h.pin_memory()
    got = P.summarize(h, w, card)
    torch.cuda.synchronize()
    assert got.is_cuda
    dev = P.summarize(h.cuda(), w, card)
    assert torch.equal(got, dev), "host-raw pipeline differs from the device-resident path"
    bad, _, _ = sax_mismatches(x, got.cpu().numpy(), w, card)
    assert len(bad) == 0, bad[:10]


def test_summarize_host_raw_default_chunk(P):
    """Default 256 MB chunks: more than one chunk at len 256 (262144 series per chunk)."""
    import torch
    n = 262_144 * 2 + 77
    x = datagen.random_walks(n, 256, 404)
    h = torch.from_numpy(x).pin_memory()
    got = P.summarize(h, 16, 256)
    dev = P.summarize(h.cuda(), 16, 256)
    assert torch.equal(got, dev)
    rows = np.r_[0:64, 262_100:262_200, n - 100:n]
    bad, _, _ = sax_mismatches(x[rows], got.cpu().numpy()[:, rows], 16, 256)
    assert len(bad) == 0, bad[:10]


@pytest.mark.parametrize("mode", ["flat", "index", "nb"])
@pytest.mark.parametrize("k", [1, 5])
def test_knn_pinned_raw(P, mode, k):
    import torch
    if mode == "nb" and k != 1:
        pytest.skip("nb-ParIS+ is 1-NN")
    n, length, nq = 40_000, 256, 24
    x = datagen.random_walks(n, length, 77 + k)
    q = datagen.random_walks(nq, length, 78 + k)
    q[:4] = x[[5, 17, 39_999, 20_000]] + 0.01 * np.random.default_rng(1).standard_normal((4, length)).astype(np.float32)
    xd = torch.from_numpy(x).cuda()
    xh = torch.from_numpy(x).pin_memory()
    sax = P.summarize(xd, 16, 256)
    qd = torch.from_numpy(q).cuda()
    if mode == "flat":
        run = lambda raw: P.knn_exact(raw, sax, qd, k=k)
    elif mode == "index":
        idx = P.index_build(sax, 16, 256)
        run = lambda raw: P.knn_index(raw, idx, qd, k=k)
    else:
        run = lambda raw: P.knn_nb(raw, sax, qd)
    hi, hd = run(xh)
    di, dd = run(xd)
    assert torch.equal(hi, di) and torch.equal(hd, dd), "pinned-raw results differ from device-raw"
    ri, rd2 = oracle.knn_bruteforce(x, q, k)
    check_knn(x, q, hi.cpu().numpy(), hd.cpu().numpy(), ri, rd2)


def test_knn_pageable_raw_rejected(P):
    import torch
    x = datagen.random_walks(64, 256, 5)
    xd = torch.from_numpy(x).cuda()
    sax = P.summarize(xd, 16, 256)
    with pytest.raises(ValueError):
        P.knn_exact(torch.from_numpy(x), sax, xd[:2])
    # the C ABI itself: pageable raw -> PARIS_EINVAL with a message
    lib = P._binding.load()
    xh = torch.from_numpy(x)
    oi = torch.empty((2, 1), dtype=torch.int64, device="cuda")
    od = torch.empty((2, 1), dtype=torch.float32, device="cuda")
    rc = lib.paris_knn_exact(xh.data_ptr(), sax.data_ptr(), 64, xd.data_ptr(), 2, 1, oi.data_ptr(),
                             od.data_ptr(), 256, 16, 256, ctypes.c_void_p(0))
    assert rc == -1 and b"page-locked" in lib.paris_last_error()
    # a host SAX array is rejected too (TMA reads it)
    sax_h = sax.cpu()
    rc = lib.paris_knn_exact(xd.data_ptr(), sax_h.data_ptr(), 64, xd.data_ptr(), 2, 1, oi.data_ptr(),
                             od.data_ptr(), 256, 16, 256, ctypes.c_void_p(0))
    assert rc == -1


@pytest.mark.parametrize("k", [1, 3])
def test_knn_index_pinned_raw_bf16(P, k):
    """Raw in pinned host memory with its bf16 copy in HBM (paris_knn_index_x): the seed's
    distances are bf16 upper bounds and the pre-filter keeps almost every fp32 row off PCIe;
    results identical to the device-raw run and the oracle (k > 1 ignores the copy)."""
    import torch
    n, length, nq = 40_000, 256, 30
    x = datagen.random_walks(n, length, 91 + k)
    q = datagen.random_walks(nq, length, 92 + k)
    q[:3] = x[[4, 30_000, 39_999]]
    xd = torch.from_numpy(x).cuda()
    xh = torch.from_numpy(x).pin_memory()
    sax = P.summarize(xd, 16, 256)
    idx = P.index_build(sax, 16, 256)
    r16 = P.raw_bf16(xd)
    qd = torch.from_numpy(q).cuda()
    hi, hd, st = P.knn_index(xh, idx, qd, k=k, raw16=r16, stats=True)
    di, dd = P.knn_index(xd, idx, qd, k=k)
    assert torch.equal(hi, di) and torch.equal(hd, dd)
    ri, rd2 = oracle.knn_bruteforce(x, q, k)
    check_knn(x, q, hi.cpu().numpy(), hd.cpu().numpy(), ri, rd2)
    if k == 1:
        assert st["refined"].float().mean().item() < 50   # fp32 rows read per query


@pytest.mark.parametrize("direct_io", [False, True])
def test_summarize_file_and_mapped_search(P, small_chunks, tmp_path, direct_io):
    """Raw data in a FILE (the paper's disk setting): paris_summarize_file (pread reader thread,
    pinned triple buffer, many chunks, O_DIRECT or buffered) gives the device path's SAX array
    and bf16 copy bit for bit; the file mapped with paris_map_raw_file serves the exact search
    (zero-copy candidate rows), equal to the oracle."""
    import torch
    n, length = 3 * 1024 + 48, 256
    x = datagen.random_walks(n, length, 3131)
    q = datagen.random_walks(5, length, 3132)
    q[2] = x[n - 7]
    path = tmp_path / "raw.f32"
    header = 4096
    with open(path, "wb") as f:
        f.write(b"\0" * header)
        f.write(np.ascontiguousarray(x).tobytes())
    xd = torch.from_numpy(x).cuda()
    ref_sax = P.summarize(xd, 16, 256)
    ref16 = P.raw_bf16(xd)
    sax, r16 = P.summarize_file(str(path), n, length, 16, 256, offset=header, bf16=True, direct_io=direct_io)
    torch.cuda.synchronize()
    assert torch.equal(sax, ref_sax)
    assert torch.equal(r16, ref16)
    bad, _, _ = sax_mismatches(x, sax.cpu().numpy(), 16, 256)
    assert len(bad) == 0
    idx = P.index_build(sax, 16, 256)
    with P.MappedRaw(str(path), n, length, offset=header) as m:
        assert m.tensor.is_pinned()
        for k, raw16 in ((1, r16), (1, None), (4, None)):
            gi, gd = P.knn_index(m.tensor, idx, torch.from_numpy(q).cuda(), k=k, raw16=raw16)
            ri, rd2 = oracle.knn_bruteforce(x, q, k)
            check_knn(x, q, gi.cpu().numpy(), gd.cpu().numpy(), ri, rd2)
    with pytest.raises(P.ParisError):
        P.summarize_file(str(path), n + 1000, length, 16, 256, offset=header)   # short file


def test_summarize_file_rejects_missing(P):
    with pytest.raises(P.ParisError):
        P.summarize_file("/nonexistent/raw.f32", 100, 256)


@pytest.mark.parametrize("source", ["pinned", "file"])
def test_host_raw_host_buffers_equal_device_buffers(P, tmp_path, source):
    """With raw outside HBM (pinned host memory, or a mapped file) and the bf16 copy in HBM,
    the end-to-end call with HOST query / output buffers (pinned; staged by the library,
    asynchronous) returns exactly the rows of the device-buffer call, over many calls on one
    stream (the cached workspace reused), and both equal the oracle."""
    import torch
    n, length, nq = 200_000, 256, 100
    x = datagen.random_walks(n, length, 5151)
    q = datagen.random_walks(nq, length, 5152)
    q[7] = x[12345]
    xd = torch.from_numpy(x).cuda()
    sax = P.summarize(xd, 16, 256)
    idx = P.index_build(sax, 16, 256)
    r16 = P.raw_bf16(xd)
    del xd
    mapped = None
    if source == "pinned":
        raw = torch.from_numpy(x).pin_memory()
    else:
        path = tmp_path / "raw.f32"
        x.tofile(path)
        mapped = P.MappedRaw(str(path), n, length)
        raw = mapped.tensor
    qd = torch.from_numpy(q).cuda()
    hq = torch.from_numpy(q).pin_memory()
    di, dd = P.knn_index(raw, idx, qd, k=1, raw16=r16)
    hi = torch.empty((nq, 1), dtype=torch.int64).pin_memory()
    hd = torch.empty((nq, 1), dtype=torch.float32).pin_memory()
    for _ in range(3):
        P.knn_index(raw, idx, hq, k=1, raw16=r16, out_idx=hi, out_dist=hd, sync=False)
        torch.cuda.current_stream().synchronize()
        assert torch.equal(hi, di.cpu()) and torch.equal(hd, dd.cpu())
    ri, rd2 = oracle.knn_bruteforce(x, q, 1)
    check_knn(x, q, hi.numpy(), hd.numpy(), ri, rd2)
    if mapped is not None:
        mapped.close()
