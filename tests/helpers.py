"""Test-support helpers mirroring proj/tests/test_support.hpp:10-33."""
import numpy as np

from oracle import bcur_oracle as O


def random_matrix(rng, rows, cols):
    """test_support.hpp:10-18 — filled row by row with rng.normal()."""
    a = np.empty((rows, cols), order="F")
    for i in range(rows):
        for j in range(cols):
            a[i, j] = rng.normal()
    return a


def random_rank_k(rng, rows, cols, k):  # test_support.hpp:20-22
    return np.asfortranarray(random_matrix(rng, rows, k) @ random_matrix(rng, k, cols))


def random_orthonormal(rng, rows, k):  # test_support.hpp:25-29
    q, _ = np.linalg.qr(random_matrix(rng, rows, k))
    return np.asfortranarray(q[:, :k])


def random_partition(rng, n, max_w):  # test_leverage.cpp:29-38
    ranges, begin = [], 0
    while begin < n:
        w = min(1 + rng.below(max_w), n - begin)
        ranges.append((begin, begin + w))
        begin += w
    return O.BlockPartition(n, ranges)


def hadamard4():
    h = np.array([[1, 1, 1, 1], [1, -1, 1, -1], [1, 1, -1, -1], [1, -1, -1, 1]], dtype=np.float64)
    return h / 2.0


def max_abs_diff(a, b):
    return float(np.max(np.abs(np.asarray(a) - np.asarray(b))))
