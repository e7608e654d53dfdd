"""The packed sign counting of score_kernel (csrc/rvk_kernels.cu sign_pair /
sign_pair_count), restated on the host: one PRMT with sign replication turns
the signs of an FFMA2 pair (g.x, g.y) into the bytes (sx, sx, sy, sy), the
loop adds such words modulo 2^32, and the count of negative values is decoded
once per scoring unit. The device path itself is checked bit-exactly by the
-m gpu parity tests (upper bounds feed every winner); this pins the algebra
for every count a unit can hold (kScorePPT = 512 points: A, B <= 256).
"""
import numpy as np


def prmt_sign_pair(gx, gy):
    """prmt.b32 d, gx, gy, 0xFFBB on float32 arrays -> uint32 words."""
    sx = (np.asarray(gx, np.float32).view(np.uint32) >> 31).astype(np.uint64)
    sy = (np.asarray(gy, np.float32).view(np.uint32) >> 31).astype(np.uint64)
    return ((sx * 0x0000FFFF + sy * 0xFFFF0000) & 0xFFFFFFFF).astype(np.uint64)


def sign_pair_count(v):
    v = np.asarray(v, np.uint64) & 0xFFFFFFFF
    a = (0x100000000 - v) & 0xFFFF
    amb = ((v + a) & 0xFFFFFFFF).astype(np.int64)
    amb = np.where(amb >= 1 << 31, amb - (1 << 32), amb) >> 16
    return 2 * a.astype(np.int64) - amb


def test_decode_every_count_of_a_unit():
    a, b = np.meshgrid(np.arange(0, 257), np.arange(0, 257), indexing="ij")
    v = (65535 * a.astype(np.int64) - 65536 * b.astype(np.int64)) % (1 << 32)
    assert np.array_equal(sign_pair_count(v.astype(np.uint64)), a + b)


def test_accumulated_words_match_sign_counts():
    rng = np.random.default_rng(5)
    for _ in range(200):
        m = int(rng.integers(0, 257))  # point pairs in a unit
        g = rng.standard_normal((m, 2)).astype(np.float32)
        g[rng.random((m, 2)) < 0.1] = np.float32(np.inf)  # padded points: never counted
        g[rng.random((m, 2)) < 0.05] = np.float32(0.0)  # e^2 == t2hi: +0, not counted
        acc = int(prmt_sign_pair(g[:, 0], g[:, 1]).sum()) & 0xFFFFFFFF
        want = int(np.count_nonzero(np.signbit(g)))
        assert int(sign_pair_count(np.uint64(acc))) == want
