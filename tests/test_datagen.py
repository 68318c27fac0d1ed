"""Harness generator checks (datagen/): Philox known-answer vectors and workload shape."""
import numpy as np

import datagen


def test_philox_known_answers():
    # Random123 Philox4x32-10 known-answer vectors (Salmon et al., SC'11 reference tests).
    kat = [
        ((0, 0, 0, 0), (0, 0), (0x6627E8D5, 0xE169C58D, 0xBC57AC4C, 0x9B00DBD8)),
        ((0xFFFFFFFF,) * 4, (0xFFFFFFFF, 0xFFFFFFFF), (0x408F276D, 0x41C83B0E, 0xA20BC7C6, 0x6D5451FD)),
        ((0x243F6A88, 0x85A308D3, 0x13198A2E, 0x03707344), (0xA4093822, 0x299F31D0),
         (0xD16CFE09, 0x94FDCCEB, 0x5001E420, 0x24126EA1)),
    ]
    for ctr, key, want in kat:
        got = tuple(int(v) for v in datagen.philox4x32(*ctr, *key))
        assert got == want


def test_normals_moments_and_independence():
    z = datagen.normals(np.arange(2000, dtype=np.uint64), 256, 7, datagen.STREAM_WALK)
    assert abs(z.mean()) < 0.01 and abs(z.std() - 1) < 0.01
    z2 = datagen.normals(np.arange(2000, dtype=np.uint64), 256, 7, datagen.STREAM_NOISE)
    assert abs(np.corrcoef(z.ravel(), z2.ravel())[0, 1]) < 0.01


def test_random_walks_znormalized_and_deterministic():
    x = datagen.random_walks(300, 256, 123)
    assert x.dtype == np.float32 and x.shape == (300, 256)
    assert np.allclose(x.mean(1), 0, atol=1e-6)
    assert np.allclose(x.astype(np.float64).std(1), 1, atol=1e-6)
    assert np.array_equal(x, datagen.random_walks(300, 256, 123))
    # a slice drawn by id offset equals the same rows of the full draw (counter-based)
    assert np.array_equal(x[100:150], datagen.random_walks(50, 256, 123, first_id=100))
    # random walk: lag-1 autocorrelation of the steps' cumulative sum is high
    r = np.mean([np.corrcoef(s[:-1], s[1:])[0, 1] for s in x[:50]])
    assert r > 0.9


def test_noisy_members():
    x = datagen.random_walks(100, 128, 5)
    src = datagen.member_ids(20, 100, 6)
    assert src.min() >= 0 and src.max() < 100
    q = datagen.noisy_members(x, src, 0.05, 6)
    assert np.allclose(q.mean(1), 0, atol=1e-6)
    d = np.sqrt(((q.astype(np.float64) - x[src]) ** 2).sum(1))
    assert np.all(d < 0.05 * np.sqrt(128) * 2)


def test_config_seeds():
    assert datagen.config_seeds(4) == (200900170, 200901170)
