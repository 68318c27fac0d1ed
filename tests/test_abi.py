"""Host-side checks of the C ABI (no GPU compute): the library builds, loads, exports every
symbol include/paris.h declares, validates arguments, and its breakpoints agree with the
oracle's independent ones.  The oracle-only boundary is also checked statically."""
import ctypes
import os
import re

import numpy as np
import pytest

import __graft_entry__ as ge

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.fixture(scope="module")
def lib():
    ge.build()
    import paper_2009_00166_b200 as p
    return p


def test_exports_every_declared_symbol(lib):
    names = lib.symbols()
    assert {"paris_summarize", "paris_knn_exact", "paris_last_error"} <= set(names)
    so = ctypes.CDLL(lib.library_path())
    for s in names:
        assert hasattr(so, s), s


def test_version_and_error_text(lib):
    assert lib.version() >= 100
    assert isinstance(lib.last_error(), str)


def test_argument_validation_without_gpu(lib):
    so = lib.load()
    # null raw -> EINVAL
    assert so.paris_summarize(None, 10, 256, 16, 256, None, None) == lib.PARIS_EINVAL
    # w does not divide len -> ECONFIG (checked before any device work)
    buf = ctypes.create_string_buffer(64)
    addr = ctypes.addressof(buf)
    assert so.paris_summarize(addr, 10, 256, 15, 256, addr, None) == lib.PARIS_ECONFIG
    assert "unsupported" in lib.last_error()
    # card not a power of two -> ECONFIG
    assert so.paris_summarize(addr, 10, 256, 16, 100, addr, None) == lib.PARIS_ECONFIG
    # k > n -> EINVAL
    assert so.paris_knn_exact(addr, addr, 5, addr, 1, 6, addr, addr, 256, 16, 256, None) == lib.PARIS_EINVAL
    assert so.paris_knn_exact(addr, addr, 5000, addr, 1, 6000, addr, addr, 256, 16, 256, None) == lib.PARIS_EINVAL
    assert so.paris_knn_approx(addr, addr, 5000, addr, 1, 2000, addr, addr, 256, 16, 256, None, None) == lib.PARIS_EINVAL
    assert so.paris_knn_exact(addr, addr, 5, addr, 1, 0, addr, addr, 256, 16, 256, None) == lib.PARIS_EINVAL
    # approximate search: same size checks
    assert so.paris_knn_approx(addr, addr, 5, addr, 1, 6, addr, addr, 256, 16, 256, None, None) == lib.PARIS_EINVAL
    # file-backed raw: null path, unsupported shape, unaligned mapping offset
    assert so.paris_summarize_file(None, 0, 10, 256, 16, 256, addr, None, 0, None) == lib.PARIS_EINVAL
    assert so.paris_summarize_file(b"/tmp/x", 0, 10, 256, 15, 256, addr, None, 0, None) == lib.PARIS_ECONFIG
    out = ctypes.c_void_p()
    assert so.paris_map_raw_file(b"/tmp/x", 17, 4096, ctypes.byref(out)) == lib.PARIS_EINVAL
    assert so.paris_map_raw_file(b"/nonexistent/raw.f32", 0, 4096, ctypes.byref(out)) == lib.PARIS_EINVAL


@pytest.mark.parametrize("card", [2, 4, 8, 16, 32, 64, 128, 256])
def test_library_breakpoints_match_oracle(lib, card):
    import oracle
    a = lib.debug_cuts(card)
    b = oracle.cuts(card)
    assert np.max(np.abs(a - b)) < 4e-15


def test_product_path_does_not_touch_oracle():
    """The package and its CUDA sources never import/include/link the oracle."""
    pkg = os.path.join(ROOT, "paper_2009_00166_b200")
    for dirpath, _, files in os.walk(pkg):
        for f in files:
            if f.endswith((".py", ".cu", ".cuh", ".h", ".cpp")):
                txt = open(os.path.join(dirpath, f)).read()
                assert not re.search(r"^\s*(import|from)\s+oracle", txt, re.M), f
                assert "liboracle" not in txt and "oracle.c" not in txt, f
    for f in os.listdir(os.path.join(ROOT, "include")):
        assert "oracle" not in open(os.path.join(ROOT, "include", f)).read().lower()


def test_missing_extension_fails_loudly(tmp_path, monkeypatch):
    import paper_2009_00166_b200._binding as b
    monkeypatch.setattr(b, "_LIBPATH", str(tmp_path / "nope.so"))
    monkeypatch.setattr(b, "_lib", None)
    with pytest.raises(b.ParisError):
        b.load()


def test_half_directed_rounding(lib):
    """The fp16 region bounds of the batched LB are rounded outward: check the library's
    directed fp16 rounding against numpy's binary16 on random, tiny, huge and exact values."""
    rng = np.random.default_rng(1)
    vals = np.concatenate([rng.normal(0, 3, 3000), rng.normal(0, 1e-5, 500),
                           rng.uniform(-7e4, 7e4, 500), [0.0, 1.0, -1.0, 65504.0, -65504.0,
                                                         2.0 ** -24, 2.0 ** -14, 6.1e-5, 0.1, -0.1]])
    for v in vals:
        dn = np.array([lib.debug_half_dir(v, -1)], dtype=np.uint16).view(np.float16)[0]
        up = np.array([lib.debug_half_dir(v, +1)], dtype=np.uint16).view(np.float16)[0]
        assert float(dn) <= v <= float(up), (v, dn, up)
        if np.isfinite(dn) and np.isfinite(up):
            # adjacent (or equal when v is representable)
            if float(dn) == v:
                assert float(up) == v
            else:
                assert np.nextafter(dn, np.float16(np.inf)) == up, (v, dn, up)
    assert np.isinf(np.array([lib.debug_half_dir(1e6, +1)], np.uint16).view(np.float16)[0])
    assert np.array([lib.debug_half_dir(1e6, -1)], np.uint16).view(np.float16)[0] == np.float16(65504)
