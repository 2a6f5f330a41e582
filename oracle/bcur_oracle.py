"""CPU oracle for the Block-CUR hot path — TEST INFRASTRUCTURE ONLY.

This module is the parity checker.  Only ``tests/``, ``__graft_entry__.smoke()``
and the ``cpu_baseline`` / ``--impl reference`` legs of ``bench.py`` may import
it.  The product (``paper_1703_06065_b200``) never imports, links or executes
anything under ``oracle/``; its compute path is the sm_100a CUDA library.

It is a numpy restatement (fp64 throughout) of the reference's algorithm for
the hot path, plus the three pieces the north star adds and the reference does
not have (randomized range finder, greedy deterministic selection, ``U=C⁺AR⁺``
with row blocks).  Every function cites the reference file:line it follows;
all reference paths are relative to ``/root/reference/proj``.

Pinning:
  * ``Rng`` is checked bit-for-bit against the reference's own ``rng.hpp``
    compiled by ``oracle/Makefile`` into ``oracle/_ref/rng_dump`` and against the
    C++ standard's known answer for ``mt19937_64``.
  * Scores, sampling, materialization, CSS and residual semantics are checked
    against every known-answer / property test the reference holds for this
    path (ported in ``tests/test_oracle_*.py``), and against a literal
    exact-SVD/pinv restatement (``reference_block_css``) on small inputs.
  * The reference's numerical core (Eigen >= 3.3, un-vendored, absent here)
    cannot be built, so there are no reference-produced golden vectors; the
    goldens in ``tests/golden/`` are produced by this oracle (script committed).
"""
from __future__ import annotations

import math
from dataclasses import dataclass, field
from typing import List, Optional, Sequence, Tuple

import numpy as np

MASK64 = (1 << 64) - 1

# ----------------------------------------------------------------------------
# Error taxonomy — errors.hpp:9-57
# ----------------------------------------------------------------------------


class Error(RuntimeError):
    """errors.hpp:10 ``Error``."""


class IterationFailure(Error):
    pass


class InvalidBasis(Error):
    pass


class ZeroBlock(Error):
    pass


class ZeroMatrix(Error):
    pass


class DistributionInvalid(Error):
    pass


class NotEnoughBlocks(Error):
    pass


class DegenerateR(Error):
    pass


class ParseError(Error):
    pass


class DimensionMismatch(Error):
    pass


# ----------------------------------------------------------------------------
# Rng — rng.hpp:13-63 (std::mt19937_64 + hand-written conversions)
# ----------------------------------------------------------------------------


class MT19937_64:
    """std::mt19937_64 (C++ [rand.predef]: w=64 n=312 m=156 r=31 ...)."""

    N, M = 312, 156
    MATRIX_A = 0xB5026F5AA96619E9
    UPPER, LOWER = 0xFFFFFFFF80000000, 0x7FFFFFFF

    def __init__(self, seed: int):
        mt = [0] * self.N
        mt[0] = seed & MASK64
        for i in range(1, self.N):
            mt[i] = (6364136223846793005 * (mt[i - 1] ^ (mt[i - 1] >> 62)) + i) & MASK64
        self.mt = mt
        self.idx = self.N

    def _twist(self):
        mt, N, M = self.mt, self.N, self.M
        for i in range(N):
            x = (mt[i] & self.UPPER) | (mt[(i + 1) % N] & self.LOWER)
            xa = x >> 1
            if x & 1:
                xa ^= self.MATRIX_A
            mt[i] = mt[(i + M) % N] ^ xa
        self.idx = 0

    def __call__(self) -> int:
        if self.idx >= self.N:
            self._twist()
        y = self.mt[self.idx]
        self.idx += 1
        y ^= (y >> 29) & 0x5555555555555555
        y ^= (y << 17) & 0x71D67FFFEDA60000
        y ^= (y << 37) & 0xFFF7EEE000000000
        y ^= y >> 43
        return y & MASK64


class Rng:
    """rng.hpp:13-63."""

    def __init__(self, seed: int):
        self._seed = seed & MASK64
        self._engine = MT19937_64(self._seed)
        self._spare = 0.0
        self._has_spare = False

    def seed(self) -> int:
        return self._seed

    def next_u64(self) -> int:
        return self._engine()

    def uniform01(self) -> float:  # rng.hpp:22
        return float(self.next_u64() >> 11) * (2.0 ** -53)

    def below(self, bound: int) -> int:  # rng.hpp:25-32
        limit = (bound * (MASK64 // bound)) & MASK64
        x = self.next_u64()
        while x >= limit:
            x = self.next_u64()
        return x % bound

    def normal(self) -> float:  # rng.hpp:35-47
        if self._has_spare:
            self._has_spare = False
            return self._spare
        u1 = 1.0 - self.uniform01()
        u2 = self.uniform01()
        radius = math.sqrt(-2.0 * math.log(u1))
        angle = 2.0 * 3.14159265358979323846 * u2
        self._spare = radius * math.sin(angle)
        self._has_spare = True
        return radius * math.cos(angle)

    def split(self, stream: int) -> "Rng":  # rng.hpp:51-56
        z = (self._seed + 0x9E3779B97F4A7C15 * (stream + 1)) & MASK64
        z = ((z ^ (z >> 30)) * 0xBF58476D1CE4E5B9) & MASK64
        z = ((z ^ (z >> 27)) * 0x94D049BB133111EB) & MASK64
        return Rng(z ^ (z >> 31))


# Stream id used to derive the sketch key from the caller's Rng without
# advancing it (the reference's Rng& contract: one uniform per draw,
# sampler.cpp:36).  Shared with the product (include/bcur_b200.h).
OMEGA_SPLIT_STREAM = 0x6F6D656761  # "omega"


def omega_key_from_seed(seed: int) -> int:
    return Rng(seed).split(OMEGA_SPLIT_STREAM).seed()


# ----------------------------------------------------------------------------
# Philox4x32-10 counter RNG (Salmon et al. 2011) — sketch Ω and generators.
# No reference counterpart (the reference sketches nothing).
# ----------------------------------------------------------------------------

PHILOX_M0, PHILOX_M1 = 0xD2511F53, 0xCD9E8D57
PHILOX_W0, PHILOX_W1 = 0x9E3779B9, 0xBB67AE85

STREAM_OMEGA = 0x4F4D4547
STREAM_U, STREAM_V, STREAM_E = 1, 2, 3
STREAM_WALK, STREAM_LOAD, STREAM_PHASE = 4, 5, 6


def philox4x32(key: int, c0, c1, c2, c3):
    """Vectorised Philox4x32-10. Inputs are uint32-valued arrays/ints."""
    u32 = np.uint64(0xFFFFFFFF)
    c0 = np.asarray(c0, dtype=np.uint64) & u32
    c1 = np.asarray(c1, dtype=np.uint64) & u32
    c2 = np.asarray(c2, dtype=np.uint64) & u32
    c3 = np.asarray(c3, dtype=np.uint64) & u32
    c0, c1, c2, c3 = np.broadcast_arrays(c0, c1, c2, c3)
    c0, c1, c2, c3 = c0.copy(), c1.copy(), c2.copy(), c3.copy()
    k0 = key & 0xFFFFFFFF
    k1 = (key >> 32) & 0xFFFFFFFF
    m0, m1 = np.uint64(PHILOX_M0), np.uint64(PHILOX_M1)
    for _ in range(10):
        p0 = m0 * c0
        p1 = m1 * c2
        hi0, lo0 = p0 >> np.uint64(32), p0 & u32
        hi1, lo1 = p1 >> np.uint64(32), p1 & u32
        n0 = hi1 ^ c1 ^ np.uint64(k0)
        n2 = hi0 ^ c3 ^ np.uint64(k1)
        c0, c1, c2, c3 = n0, lo1, n2, lo0
        k0 = (k0 + PHILOX_W0) & 0xFFFFFFFF
        k1 = (k1 + PHILOX_W1) & 0xFFFFFFFF
    return c0, c1, c2, c3


def omega(n: int, l: int, key: int) -> np.ndarray:
    """Rademacher sketch Ω (n×l, ±1 fp64).

    Ω[j, c] = 1 − 2·bit(c mod 128) of Philox(key, (j_lo, j_hi, c div 128, STREAM_OMEGA)).
    """
    j = np.arange(n, dtype=np.uint64)
    out = np.empty((n, l), dtype=np.float64, order="F")
    for grp in range((l + 127) // 128):
        w = philox4x32(key, j & np.uint64(0xFFFFFFFF), j >> np.uint64(32), grp, STREAM_OMEGA)
        for b in range(min(128, l - grp * 128)):
            bit = (w[b >> 5] >> np.uint64(b & 31)) & np.uint64(1)
            out[:, grp * 128 + b] = 1.0 - 2.0 * bit.astype(np.float64)
    return out


def gaussian(key: int, stream: int, count: int, offset: int = 0) -> np.ndarray:
    """Counter-based N(0,1): element e -> Philox(key, (e_lo, e_hi, 0, stream)), Box–Muller."""
    e = np.arange(offset, offset + count, dtype=np.uint64)
    w0, w1, w2, w3 = philox4x32(key, e & np.uint64(0xFFFFFFFF), e >> np.uint64(32), 0, stream)
    a = ((w0 << np.uint64(32)) | w1) >> np.uint64(11)
    b = ((w2 << np.uint64(32)) | w3) >> np.uint64(11)
    u1 = 1.0 - a.astype(np.float64) * (2.0 ** -53)  # (0, 1]
    u2 = b.astype(np.float64) * (2.0 ** -53)
    return np.sqrt(-2.0 * np.log(u1)) * np.cos(2.0 * math.pi * u2)


def uniform(key: int, stream: int, count: int) -> np.ndarray:
    e = np.arange(count, dtype=np.uint64)
    w0, w1, _, _ = philox4x32(key, e & np.uint64(0xFFFFFFFF), e >> np.uint64(32), 0, stream)
    a = ((w0 << np.uint64(32)) | w1) >> np.uint64(11)
    return a.astype(np.float64) * (2.0 ** -53)


# ----------------------------------------------------------------------------
# Synthetic inputs.  Reference shape/RNG-order analogue:
# synthetic_low_rank, bench.cpp:11-39 (which uses un-orthonormalised factors).
# ----------------------------------------------------------------------------


def orthonormal_factor(x: np.ndarray) -> np.ndarray:
    """Orthonormal basis with positive R diagonal (canonical; matches CholQR)."""
    q, r = np.linalg.qr(x)
    d = np.sign(np.diag(r))
    d[d == 0] = 1.0
    return np.asfortranarray(q * d)


def gen_lowrank(m: int, n: int, sigma: Sequence[float], noise: float, seed: int,
                dtype=np.float64) -> np.ndarray:
    """A = U·diag(σ)·Vᵀ + ν·E, U,V Gaussian-then-orthonormalised (column-major)."""
    r = len(sigma)
    u0 = gaussian(seed, STREAM_U, m * r).reshape((m, r), order="F")
    v0 = gaussian(seed, STREAM_V, n * r).reshape((n, r), order="F")
    u = orthonormal_factor(u0) * np.asarray(sigma, dtype=np.float64)[None, :]
    v = orthonormal_factor(v0)
    a = np.zeros((m, n), dtype=np.float64, order="F")
    for t in range(r):  # fixed-order accumulation, no fma
        a += np.outer(u[:, t], v[:, t])
    if noise > 0.0:
        a += noise * gaussian(seed, STREAM_E, m * n).reshape((m, n), order="F")
    return np.asfortranarray(a.astype(dtype))


def gen_biometric(m: int, n: int, seed: int, walk_sigma: float = 0.05, window: int = 50,
                  n_trends: int = 5) -> np.ndarray:
    """Config-2 shape: smoothed random walks + rank-5 shared trends (fp64).

    x_i = MA_window(cumsum(walk_sigma·ε_i)) + Σ_t L[i,t]·cos(2π(t+1)j/n + φ_t)
    (trailing moving average; partial windows at the start).
    """
    inc = walk_sigma * gaussian(seed, STREAM_WALK, m * n).reshape((m, n), order="F")
    walk = np.cumsum(inc, axis=1)
    cs = np.concatenate([np.zeros((m, 1)), np.cumsum(walk, axis=1)], axis=1)
    j = np.arange(n)
    lo = np.maximum(j + 1 - window, 0)
    ma = (cs[:, j + 1] - cs[:, lo]) / (j + 1 - lo)[None, :]
    load = gaussian(seed, STREAM_LOAD, m * n_trends).reshape((m, n_trends), order="F")
    phase = 2.0 * math.pi * uniform(seed, STREAM_PHASE, n_trends)
    trends = np.stack([np.cos(2.0 * math.pi * (t + 1) * j / n + phase[t]) for t in range(n_trends)], axis=1)
    return np.asfortranarray(ma + load @ trends.T)


# ----------------------------------------------------------------------------
# Partitions — leverage.cpp:27-90
# ----------------------------------------------------------------------------


class BlockPartition:
    def __init__(self, n: int, ranges: Sequence[Tuple[int, int]]):
        if n < 1:
            raise ValueError("BlockPartition: n must be >= 1")
        if len(ranges) == 0:
            raise ValueError("BlockPartition: at least one block required")
        expect = 0
        for b, e in ranges:
            if b != expect or e <= b:
                raise ValueError("BlockPartition: ranges must be contiguous, non-empty, and ordered")
            expect = e
        if expect != n:
            raise ValueError("BlockPartition: ranges must cover [0, n) exactly")
        self.n = n
        self.ranges = [(int(b), int(e)) for b, e in ranges]
        self.nominal = self.max_width()

    @staticmethod
    def equal_blocks(n: int, s: int) -> "BlockPartition":  # leverage.cpp:29-41
        if n < 1 or s < 1:
            raise ValueError("equal_blocks: n and block_size must be >= 1")
        p = BlockPartition(n, [(b, min(b + s, n)) for b in range(0, n, s)])
        p.nominal = s
        return p

    @staticmethod
    def from_boundaries(n: int, cuts: Sequence[int]) -> "BlockPartition":  # leverage.cpp:43-56
        ranges, begin = [], 0
        for c in cuts:
            if c <= begin or c >= n:
                raise ValueError("from_boundaries: cuts must be strictly increasing and inside (0, n)")
            ranges.append((begin, c))
            begin = c
        ranges.append((begin, n))
        return BlockPartition(n, ranges)

    def num_blocks(self) -> int:
        return len(self.ranges)

    def max_width(self) -> int:
        return max(e - b for b, e in self.ranges)

    def width(self, g: int) -> int:
        b, e = self.ranges[g]
        return e - b

    def offsets(self) -> np.ndarray:
        return np.array([b for b, _ in self.ranges] + [self.n], dtype=np.int64)

    def block_of_column(self, j: int) -> int:  # leverage.cpp:82-90
        if j < 0 or j >= self.n:
            raise IndexError("block_of_column: column index out of range")
        return int(np.searchsorted(self.offsets()[:-1], j, side="right") - 1)


# ----------------------------------------------------------------------------
# Scores — leverage.cpp:11-23, 92-121
# ----------------------------------------------------------------------------

ORTHONORMAL_TOL = {np.dtype(np.float64): 1e-8, np.dtype(np.float32): 1e-4}


def require_orthonormal(v: np.ndarray, tol: float = 1e-8, what: str = "basis") -> float:
    """leverage.cpp:11-23 (tolerance dtype-aware per SURVEY D13)."""
    if v.ndim != 2 or v.shape[0] < 1 or v.shape[1] < 1:
        raise InvalidBasis(f"{what}: basis must be non-empty")
    if v.shape[0] < v.shape[1]:
        raise InvalidBasis(f"{what}: more columns than rows cannot be orthonormal")
    v64 = v.astype(np.float64)
    dev = float(np.max(np.abs(v64.T @ v64 - np.eye(v.shape[1]))))
    if dev > tol:
        raise InvalidBasis(f"{what}: column Gram deviates from identity by {dev}")
    return dev


@dataclass
class ScoreVector:
    scores: np.ndarray
    normalizer: float = 1.0

    def probabilities(self) -> np.ndarray:
        return self.scores / self.normalizer

    def distribution(self) -> np.ndarray:  # leverage.cpp:92-98
        total = float(np.sum(self.scores))
        if not total > 0.0:
            raise ZeroMatrix("ScoreVector::distribution: scores sum to zero")
        return self.scores / total


def column_leverage(v_k: np.ndarray, tol: float = 1e-8) -> ScoreVector:  # leverage.cpp:100-106
    require_orthonormal(v_k, tol, "column_leverage")
    v = v_k.astype(np.float64)
    return ScoreVector(np.sum(v * v, axis=1), float(v.shape[1]))


def block_sums(row_values: np.ndarray, part: BlockPartition) -> np.ndarray:
    off = part.offsets()
    return np.array([float(np.sum(row_values[off[g]:off[g + 1]])) for g in range(len(off) - 1)])


def block_leverage(v_k: np.ndarray, part: BlockPartition, tol: float = 1e-8,
                   check: bool = True) -> ScoreVector:  # leverage.cpp:108-121
    if check:
        require_orthonormal(v_k, tol, "block_leverage")
    if v_k.shape[0] != part.n:
        raise DimensionMismatch("block_leverage: partition size does not match V_k rows")
    v = v_k.astype(np.float64)
    return ScoreVector(block_sums(np.sum(v * v, axis=1), part), float(v.shape[1]))


# ----------------------------------------------------------------------------
# Sampling — sampler.cpp:16-50, 116-202
# ----------------------------------------------------------------------------

WITH_REPLACEMENT = "with_replacement"
WITHOUT_REPLACEMENT = "without_replacement"


@dataclass
class BlockDraw:
    block: int
    probability: float
    scale: float


@dataclass
class SamplingPlan:
    draws: List[BlockDraw]
    mode: str = WITH_REPLACEMENT
    seed: int = 0
    margins: List[float] = field(default_factory=list)  # D14 near-tie record

    def blocks(self) -> List[int]:
        return [d.block for d in self.draws]


def require_distribution(probs: np.ndarray) -> None:  # sampler.cpp:16-31
    if probs.size < 1:
        raise DistributionInvalid("empty probability vector")
    s = 0.0
    for i, p in enumerate(probs):
        if not math.isfinite(p) or p < 0.0:
            raise DistributionInvalid(f"probability {i} is negative or non-finite")
        s += p
    if abs(s - 1.0) > 1e-10:
        raise DistributionInvalid(f"probabilities sum to {s}, not 1")


def categorical_draw(probs, active, mass, rng: Rng):  # sampler.cpp:35-50
    """Returns (index, margin) — margin = distance of u to the nearest CDF edge."""
    u = rng.uniform01() * mass
    cum = 0.0
    last_positive = -1
    prev = 0.0
    for i in range(len(probs)):
        if not active[i] or probs[i] <= 0.0:
            continue
        last_positive = i
        prev = cum
        cum += probs[i]
        if cum > u:
            return i, min(u - prev, cum - u)
    return last_positive, 0.0


def draw_blocks(probs: np.ndarray, g: int, mode: str, rng: Rng) -> SamplingPlan:  # sampler.cpp:116-146
    if g < 1:
        raise ValueError("draw_blocks: g must be >= 1")
    probs = np.asarray(probs, dtype=np.float64)
    require_distribution(probs)
    plan = SamplingPlan([], mode, rng.seed())
    active = [True] * probs.size
    if mode == WITHOUT_REPLACEMENT:
        positive = int(np.sum(probs > 0.0))
        if g > positive:
            raise NotEnoughBlocks(f"draw_blocks: asked for {g} distinct blocks but only {positive} have positive probability")
    mass = 1.0
    for _ in range(g):
        j, margin = categorical_draw(probs, active, mass, rng)
        p = float(probs[j])
        plan.draws.append(BlockDraw(j, p, 1.0 / math.sqrt(g * p)))
        plan.margins.append(margin)
        if mode == WITHOUT_REPLACEMENT:
            active[j] = False
            mass -= p
    return plan


def identity_plan(part: BlockPartition) -> SamplingPlan:  # sampler.cpp:148-159
    G = part.num_blocks()
    return SamplingPlan([BlockDraw(j, 1.0 / G, 1.0) for j in range(G)], WITHOUT_REPLACEMENT, 0)


def materialize_columns(a: np.ndarray, part: BlockPartition, plan: SamplingPlan) -> np.ndarray:
    """sampler.cpp:161-184."""
    if a.shape[1] != part.n:
        raise DimensionMismatch("materialize_columns: A columns do not match partition")
    if not plan.draws:
        raise ValueError("materialize_columns: empty plan")
    cols = []
    for d in plan.draws:
        if d.block < 0 or d.block >= part.num_blocks():
            raise DimensionMismatch(f"materialize_columns: plan references block {d.block} outside the partition")
        b, e = part.ranges[d.block]
        cols.append(cols64(a, b, e) * d.scale)
    return np.asfortranarray(np.concatenate(cols, axis=1))


def materialize_row_blocks(a: np.ndarray, part: BlockPartition, plan: SamplingPlan) -> np.ndarray:
    """Row blocks = column blocks of Aᵀ; sampler.cpp:186-202 analogue."""
    return np.asfortranarray(materialize_columns(a.T, part, plan).T)


# ----------------------------------------------------------------------------
# Dense helpers — matcore.cpp:35-110 semantics where a reference item exists
# ----------------------------------------------------------------------------


def rank_tolerance(rows: int, cols: int, sigma_max: float) -> float:  # matcore.cpp:35-37
    return 1e-12 * max(rows, cols) * sigma_max


# Products with A in fp64.  An fp32 A (configs c3–c5) is converted column chunk by column
# chunk (exactly: fp32 ⊂ fp64) instead of as a whole, which only bounds host memory — the
# full-size parity tests hold c3/c4's A (4.3 GB fp32; its fp64 copy alone would be 8.6 GB).
# fp64 inputs take the direct products (bit-identical to the committed c1/c2 goldens).
CHUNK_ELEMS = 1 << 26


def _chunks(a: np.ndarray):
    m, n = a.shape
    w = max(1, min(n, CHUNK_ELEMS // max(m, 1)))
    for j0 in range(0, n, w):
        yield j0, min(n, j0 + w)


def cols64(a: np.ndarray, j0: int, j1: int) -> np.ndarray:
    return np.asarray(a[:, j0:j1], dtype=np.float64)


def a_mul(a: np.ndarray, x: np.ndarray) -> np.ndarray:
    """A·x (x: n × N fp64)."""
    if a.dtype == np.float64:
        return a @ x
    out = np.zeros((a.shape[0], x.shape[1]))
    for j0, j1 in _chunks(a):
        out += cols64(a, j0, j1) @ x[j0:j1]
    return out


def at_mul(a: np.ndarray, y: np.ndarray) -> np.ndarray:
    """Aᵀ·y (y: m × N fp64) → n × N."""
    if a.dtype == np.float64:
        return a.T @ y
    out = np.empty((a.shape[1], y.shape[1]))
    for j0, j1 in _chunks(a):
        out[j0:j1] = cols64(a, j0, j1).T @ y
    return out


def col_sumsq(a: np.ndarray) -> np.ndarray:
    """Σ_i a(i, j)² per column, fp64."""
    if a.dtype == np.float64:
        return np.sum(a * a, axis=0)
    out = np.empty(a.shape[1])
    for j0, j1 in _chunks(a):
        c = cols64(a, j0, j1)
        out[j0:j1] = np.einsum("ij,ij->j", c, c)
    return out


def row_sumsq(a: np.ndarray) -> np.ndarray:
    """Σ_j a(i, j)² per row, fp64."""
    if a.dtype == np.float64:
        return np.sum(a * a, axis=1)
    out = np.zeros(a.shape[0])
    for j0, j1 in _chunks(a):
        c = cols64(a, j0, j1)
        out += np.einsum("ij,ij->i", c, c)
    return out


def resid_sumsq(a: np.ndarray, left: np.ndarray, right_t: np.ndarray) -> float:
    """‖A − left·right_tᵀ‖_F² (left: m × r, right_t: n × r), streamed over column chunks."""
    if a.dtype == np.float64:
        r = a - left @ right_t.T
        return float(np.sum(r * r))
    tot = 0.0
    for j0, j1 in _chunks(a):
        r = cols64(a, j0, j1) - left @ right_t[j0:j1].T
        tot += float(np.einsum("ij,ij->", r, r))
    return tot


# Orthonormalisation thresholds.
TAU_CHOL = {np.dtype(np.float64): 1e-5, np.dtype(np.float32): 1e-2}
TAU_RANK = {np.dtype(np.float64): 1e-7, np.dtype(np.float32): 1e-5}
THETA_EXPLICIT = {np.dtype(np.float64): 1e-6, np.dtype(np.float32): 0.1}


def right_solve_upper(x: np.ndarray, r: np.ndarray) -> np.ndarray:
    """X·R⁻¹ for upper-triangular R (a triangular solve, not an LU of R)."""
    from scipy.linalg import solve_triangular
    return solve_triangular(r, x.T, trans="T", lower=False, check_finite=False).T


def chol_upper(g: np.ndarray) -> Optional[np.ndarray]:
    try:
        return np.linalg.cholesky(g).T  # upper R, g = RᵀR
    except np.linalg.LinAlgError:
        return None


def eig_desc(g: np.ndarray):
    lam, w = np.linalg.eigh(g)
    order = np.argsort(lam)[::-1]
    return lam[order], w[:, order]


def orth(x: np.ndarray, ref: float, dt) -> Tuple[np.ndarray, np.ndarray, str]:
    """Rank-revealing orthonormalisation X ≈ Q·T (Q: m×r orthonormal, T: r×w).

    Path "chol": CholQR2 if chol(XᵀX) succeeds with min R_ii > τ_chol·ref.
    Path "eig":  SVQB (eig of XᵀX — or of X·Xᵀ for a wide panel, rows < w — keep
                 σ_i > τ_rank·ref) then one CholQR pass.
    Replaces the reference's SVD-based pinv/rank cut (matcore.cpp:39-56,85-91).
    """
    dt = np.dtype(dt)
    x = np.asarray(x, dtype=np.float64)
    w = x.shape[1]
    if w == 0:
        return np.zeros((x.shape[0], 0)), np.zeros((0, 0)), "empty"
    g = x.T @ x
    r = chol_upper(g)
    if r is not None and np.all(np.isfinite(r)) and np.min(np.diag(r)) > TAU_CHOL[dt] * ref:
        q1 = right_solve_upper(x, r)  # X R⁻¹
        r2 = chol_upper(q1.T @ q1)
        q = right_solve_upper(q1, r2)
        return q, r2 @ r, "chol"
    if x.shape[0] < w:
        # wide panel: decide on the smaller row Gram X·Xᵀ.  Safely full row rank (its
        # Cholesky passes the same τ_chol test) → range(X) = ℝ^rows, Q = I, T = X;
        # otherwise its eigenvectors are the orthonormal basis directly.
        gr = x @ x.T
        rr = chol_upper(gr)
        if rr is not None and np.all(np.isfinite(rr)) and np.min(np.diag(rr)) > TAU_CHOL[dt] * ref:
            return np.eye(x.shape[0]), x.copy(), "eig"
        lam, u = eig_desc(gr)
        sig = np.sqrt(np.maximum(lam, 0.0))
        keep = int(np.sum(sig > TAU_RANK[dt] * ref))
        if keep == 0:
            return np.zeros((x.shape[0], 0)), np.zeros((0, w)), "eig"
        q1 = u[:, :keep]
        r2 = chol_upper(q1.T @ q1)
        q = right_solve_upper(q1, r2)
        return q, r2 @ (q1.T @ x), "eig"
    lam, wv = eig_desc(g)
    sig = np.sqrt(np.maximum(lam, 0.0))
    keep = int(np.sum(sig > TAU_RANK[dt] * ref))
    if keep == 0:
        return np.zeros((x.shape[0], 0)), np.zeros((0, w)), "eig"
    q1 = (x @ wv[:, :keep]) / sig[:keep]
    r2 = chol_upper(q1.T @ q1)
    q = right_solve_upper(q1, r2)
    t = (r2 * sig[:keep][None, :]) @ wv[:, :keep].T
    return q, t, "eig"


def cgs2_panel(qc: np.ndarray, p: np.ndarray, ref: float, dt):
    """Block classical Gram–Schmidt, two passes, then rank-revealing orth."""
    coef = np.zeros((qc.shape[1], p.shape[1]))
    if qc.shape[1] > 0:
        for _ in range(2):
            x = qc.T @ p
            p = p - qc @ x
            coef += x
    q, t, path = orth(p, ref, dt)
    return q, coef, t, path


# ----------------------------------------------------------------------------
# N1: randomized range finder (no reference; "sketching")
# ----------------------------------------------------------------------------


@dataclass
class Subspace:
    v_k: np.ndarray        # n × k_eff right singular vectors
    u_k: np.ndarray        # m × k_eff left singular vectors
    sigma: np.ndarray      # sketch singular values (all r kept)
    k_eff: int
    l: int
    q_rank: int


def range_finder(a: np.ndarray, k: int, p: int, q: int, key: int, rank_floor: bool = False) -> Subspace:
    """Y = AΩ, q power iterations, Q = orth(Y), Bᵀ = AᵀQ, eig of BBᵀ, V_k = BᵀŨ_kΣ_k⁻¹.

    The numerical rank of the sketch is the reference's (matcore.cpp:35-49: σ >
    1e-12·max(m,n)·σ₁).  rank_floor=True (opt-in) also drops σ ≤ τ_rank·σ₁ (1e-7 fp64,
    1e-5 fp32): directions below the working precision of an fp32 A.
    """
    dt = np.dtype(a.dtype)
    if dt not in (np.dtype(np.float32), np.dtype(np.float64)):
        a = np.asarray(a, dtype=np.float64)
        dt = a.dtype
    m, n = a.shape
    l = min(k + p, m, n)
    om = omega(n, l, key)
    y = a_mul(a, om)
    for _ in range(q):
        qy, _, _ = orth(y, float(np.sqrt(np.max(np.sum(y * y, axis=0)))), dt)
        z = at_mul(a, qy)
        qz, _, _ = orth(z, float(np.sqrt(np.max(np.sum(z * z, axis=0)))), dt)
        y = a_mul(a, qz)
    qy, _, _ = orth(y, float(np.sqrt(np.max(np.sum(y * y, axis=0)))), dt)
    bt = at_mul(a, qy)                # n × r  (B = Qᵀ A)
    lam, ut = eig_desc(bt.T @ bt)     # B Bᵀ
    sig = np.sqrt(np.maximum(lam, 0.0))
    if sig.size == 0 or not sig[0] > 0.0:
        raise ZeroMatrix("range_finder: A is identically zero")
    tol = rank_tolerance(m, n, sig[0])
    if rank_floor:
        tol = max(tol, TAU_RANK[dt] * sig[0])
    rank = int(np.sum(sig > tol))
    k_eff = min(k, rank)
    wmat = ut[:, :k_eff] / sig[:k_eff]
    v_k = bt @ wmat
    u_k = qy @ ut[:, :k_eff]
    return Subspace(v_k, u_k, sig[:rank], k_eff, l, qy.shape[1])


def exact_subspace(a: np.ndarray, k: int) -> Subspace:
    """Reference semantics: truncate(svd(a), k) (matcore.cpp:39-69)."""
    a = np.asarray(a, dtype=np.float64)
    u, s, vt = np.linalg.svd(a, full_matrices=False)
    tol = rank_tolerance(a.shape[0], a.shape[1], s[0]) if s.size else 0.0
    rank = int(np.sum((s > tol) & (s > 0)))
    keep = min(k, rank)
    return Subspace(vt[:keep].T.copy(), u[:, :keep].copy(), s[:rank], keep, keep, rank)


# ----------------------------------------------------------------------------
# Factor construction + residual (R14/R15/N4)
# ----------------------------------------------------------------------------


def unique_in_order(blocks: Sequence[int]) -> List[int]:
    seen, out = set(), []
    for b in blocks:
        if b not in seen:
            seen.add(b)
            out.append(b)
    return out


def cholqr2_whole(c: np.ndarray, dt) -> Optional[np.ndarray]:
    """Whole-C CholQR2 when C is safely full rank: chol(CᵀC) succeeds with
    min R_ii > τ_chol · max_j ‖c_j‖ (the same test the GPU applies before taking
    its tensor-core path); None → fall back to block CGS2 panels."""
    if c.shape[1] == 0:
        return None
    g = c.T @ c
    r = chol_upper(g)
    ref = float(np.sqrt(np.max(np.diag(g))))
    if r is None or not np.all(np.isfinite(r)) or not np.min(np.diag(r)) > TAU_CHOL[np.dtype(dt)] * ref:
        return None
    q1 = right_solve_upper(c, r)
    r2 = chol_upper(q1.T @ q1)
    if r2 is None:
        return None
    return right_solve_upper(q1, r2)


def column_basis(a64: np.ndarray, part: BlockPartition, blocks: Sequence[int], dt,
                 block_norms: np.ndarray, allow_whole: bool = True):
    """Q_C for the unique selected blocks (draw order): whole-C CholQR2 when safely
    full rank, else block CGS2 panels with per-panel rank revealing."""
    m = a64.shape[0]
    ub = unique_in_order(blocks)
    if allow_whole:
        cols = np.concatenate([cols64(a64, *part.ranges[b]) for b in ub], axis=1)
        q = cholqr2_whole(cols, dt)
        if q is not None:
            return q, ["whole"]
    qc = np.zeros((m, 0))
    paths = []
    for bidx in ub:
        b, e = part.ranges[bidx]
        ref = math.sqrt(block_norms[bidx])
        qn, _, _, path = cgs2_panel(qc, cols64(a64, b, e).copy(), ref, dt)
        qc = np.concatenate([qc, qn], axis=1)
        paths.append(path)
    return qc, paths


def projection_residual(a64: np.ndarray, qc: np.ndarray, a_norm2: float, dt,
                        force: Optional[str] = None) -> Tuple[float, str]:
    """‖A − Q_C Q_Cᵀ A‖_F² — Pythagoras, explicit when small.
    force: "explicit" / "pythagoras" overrides the rule (the ABI's residual mode)."""
    xt = at_mul(a64, qc)  # (Q_Cᵀ A)ᵀ, n × r
    res2 = a_norm2 - float(np.einsum("ij,ij->", xt, xt))
    if force == "explicit" or (force is None and res2 < THETA_EXPLICIT[np.dtype(dt)] * a_norm2):
        return resid_sumsq(a64, qc, xt), "explicit"
    return max(res2, 0.0), "pythagoras"


@dataclass
class CssResult:
    plan: SamplingPlan
    scores: ScoreVector
    abs_err: float
    a_norm: float
    rank_c: int
    residual_path: str
    subspace: Optional[Subspace] = None

    @property
    def rel_err(self) -> float:
        return self.abs_err / self.a_norm if self.a_norm > 0 else 0.0


def block_norms2(a64: np.ndarray, part: BlockPartition) -> np.ndarray:
    return block_sums(col_sumsq(a64), part)


def block_css(a: np.ndarray, part: BlockPartition, k: int, g: int, rng: Rng, p: int = 5, q: int = 0,
              mode: str = WITH_REPLACEMENT, exact: bool = False, residual: Optional[str] = None,
              rank_floor: bool = False) -> CssResult:
    """sketch.cpp:68-82 with the range finder (N1) in place of the exact SVD.

    ``exact=True`` uses truncate(svd(a), k) like the reference (small inputs).
    An fp32 A is not copied to fp64 as a whole (products convert column chunks).
    """
    if k < 1:
        raise ValueError("block_css: k must be >= 1")
    if a.shape[1] != part.n:
        raise DimensionMismatch("block_css: partition does not match A columns")
    dt = a.dtype
    a64 = a if dt in (np.float32, np.float64) else np.asarray(a, dtype=np.float64)
    bn2 = block_norms2(a64, part)
    a_norm2 = float(np.sum(bn2))
    if not a_norm2 > 0.0:
        raise ZeroMatrix("block_css: A is identically zero")
    if exact:
        sub = exact_subspace(np.asarray(a, dtype=np.float64), k)
    else:
        sub = range_finder(a64, k, p, q, omega_key_from_seed(rng.seed()), rank_floor=rank_floor)
    if sub.k_eff == 0:
        raise ZeroMatrix("block_css: A is identically zero")
    scores = block_leverage(sub.v_k, part, check=False)
    plan = draw_blocks(scores.distribution(), g, mode, rng)
    qc, _ = column_basis(a64, part, plan.blocks(), dt, bn2)
    res2, path = projection_residual(a64, qc, a_norm2, dt, force=residual)
    return CssResult(plan, scores, math.sqrt(res2), math.sqrt(a_norm2), qc.shape[1], path, sub)


def reference_block_css(a: np.ndarray, part: BlockPartition, k: int, g: int, rng: Rng,
                        mode: str = WITH_REPLACEMENT) -> CssResult:
    """Literal reference semantics (sketch.cpp:68-82): exact SVD + pinv(C)."""
    a64 = np.asarray(a, dtype=np.float64)
    sub = exact_subspace(a64, k)
    scores = block_leverage(sub.v_k, part)
    plan = draw_blocks(scores.distribution(), g, mode, rng)
    c = materialize_columns(a64, part, plan)
    err = float(np.linalg.norm(a64 - c @ (pinv(c) @ a64)))
    return CssResult(plan, scores, err, float(np.linalg.norm(a64)), 0, "pinv", sub)


def pinv(a: np.ndarray) -> np.ndarray:
    """matcore.cpp:85-91 (SVD, rank_tolerance cut)."""
    u, s, vt = np.linalg.svd(a, full_matrices=False)
    if s.size == 0 or s[0] == 0.0:
        return np.zeros((a.shape[1], a.shape[0]))
    tol = rank_tolerance(a.shape[0], a.shape[1], s[0])
    r = int(np.sum((s > tol) & (s > 0)))
    return (vt[:r].T / s[:r]) @ u[:, :r].T


def error_report(a: np.ndarray, c: np.ndarray, u: np.ndarray, r: np.ndarray) -> Tuple[float, float]:
    """blockcur.cpp:33-52: (abs_err, rel_to_a) with abs = ‖A − C(UR)‖_F."""
    if c.shape[0] != a.shape[0] or r.shape[1] != a.shape[1] or u.shape[0] != c.shape[1] or u.shape[1] != r.shape[0]:
        raise DimensionMismatch("error_report: C U R shapes do not compose to the shape of A")
    a64 = np.asarray(a, dtype=np.float64)
    abs_err = float(np.linalg.norm(a64 - c.astype(np.float64) @ (u.astype(np.float64) @ r.astype(np.float64))))
    an = float(np.linalg.norm(a64))
    return abs_err, (abs_err / an if an > 0 else 0.0)


# ----------------------------------------------------------------------------
# N3: greedy deterministic selection
# ----------------------------------------------------------------------------

TAU_SATURATE = {np.dtype(np.float64): 1e-12, np.dtype(np.float32): 1e-6}


@dataclass
class GreedyStep:
    block: int
    score: float
    margin: float
    saturated: bool
    rank_added: int


@dataclass
class GreedyResult:
    steps: List[GreedyStep]
    abs_err: float
    a_norm: float
    residuals: np.ndarray
    residual_path: str

    def blocks(self) -> List[int]:
        return [s.block for s in self.steps]

    @property
    def rel_err(self) -> float:
        return self.abs_err / self.a_norm if self.a_norm > 0 else 0.0


def argmax_lowest(vals: np.ndarray, allowed: np.ndarray) -> Tuple[int, float]:
    """argmax over allowed entries, ties → lowest index; returns (index, top1−top2)."""
    idx = np.flatnonzero(allowed)
    v = vals[idx]
    best = int(idx[int(np.argmax(v))])  # np.argmax returns the first maximum
    if idx.size > 1:
        srt = np.sort(v)[::-1]
        margin = float(srt[0] - srt[1])
    else:
        margin = float("inf")
    return best, margin


def greedy_select(a: np.ndarray, part: BlockPartition, k: int, g: int, key: int, p: int = 5,
                  q: int = 0) -> GreedyResult:
    dt = np.dtype(a.dtype)
    a64 = np.asarray(a, dtype=np.float64)
    G = part.num_blocks()
    if g < 1 or g > G:
        raise ValueError("greedy_select: need 1 <= g <= number of blocks")
    bn2 = block_norms2(a64, part)
    a_norm2 = float(np.sum(bn2))
    if not a_norm2 > 0.0:
        raise ZeroMatrix("greedy_select: A is identically zero")
    res = bn2.copy()
    selected = np.zeros(G, dtype=bool)
    qc = np.zeros((a64.shape[0], 0))
    lev = None
    steps = []
    off = part.offsets()
    for _ in range(g):
        j, margin = argmax_lowest(res, ~selected)
        saturated = bool(res[j] <= TAU_SATURATE[dt] * a_norm2)
        if saturated:
            if lev is None:
                sub = range_finder(a, k, p, q, key)
                lev = block_leverage(sub.v_k, part, check=False).scores
            j, margin = argmax_lowest(lev, ~selected)
        score = float(res[j])
        selected[j] = True
        b, e = part.ranges[j]
        qn, _, _, _ = cgs2_panel(qc, a64[:, b:e].copy(), math.sqrt(bn2[j]), dt)
        if qn.shape[1] > 0:
            x = qn.T @ a64
            res = res - block_sums(np.sum(x * x, axis=0), part)
            qc = np.concatenate([qc, qn], axis=1)
        steps.append(GreedyStep(j, score, margin, saturated, qn.shape[1]))
    res2 = float(np.sum(res))
    path = "pythagoras"
    if res2 < THETA_EXPLICIT[dt] * a_norm2:
        x = qc.T @ a64
        r = a64 - qc @ x
        res2, path = float(np.sum(r * r)), "explicit"
    return GreedyResult(steps, math.sqrt(max(res2, 0.0)), math.sqrt(a_norm2), res, path)


# ----------------------------------------------------------------------------
# N4: block CUR with row and column blocks, U = C⁺ A R⁺
# ----------------------------------------------------------------------------


@dataclass
class CurResult:
    col_plan: SamplingPlan
    row_plan: SamplingPlan
    col_scores: ScoreVector
    row_scores: ScoreVector
    u: Optional[np.ndarray]
    abs_err: float
    a_norm: float
    residual_path: str

    @property
    def rel_err(self) -> float:
        return self.abs_err / self.a_norm if self.a_norm > 0 else 0.0


def block_cur_rows_cols(a: np.ndarray, col_part: BlockPartition, row_part: BlockPartition, k: int,
                        gc: int, gr: int, rng: Rng, p: int = 10, q: int = 0,
                        mode: str = WITHOUT_REPLACEMENT, want_u: bool = True, rank_floor: bool = False) -> CurResult:
    dt = np.dtype(a.dtype)
    a64 = a if dt in (np.dtype(np.float32), np.dtype(np.float64)) else np.asarray(a, dtype=np.float64)
    if col_part.n != a.shape[1] or row_part.n != a.shape[0]:
        raise DimensionMismatch("block_cur: partitions do not match A")
    a_norm2 = float(np.sum(col_sumsq(a64)))
    if not a_norm2 > 0.0:
        raise ZeroMatrix("block_cur: A is identically zero")
    sub = range_finder(a64, k, p, q, omega_key_from_seed(rng.seed()), rank_floor=rank_floor)
    cs = block_leverage(sub.v_k, col_part, check=False)
    rs = block_leverage(sub.u_k, row_part, check=False)
    cplan = draw_blocks(cs.distribution(), gc, mode, rng)
    rplan = draw_blocks(rs.distribution(), gr, mode, rng)
    qc, _ = column_basis(a64, col_part, cplan.blocks(), dt, block_norms2(a64, col_part))
    at = a64.T  # row blocks of A = column blocks of Aᵀ (a view: no copy)
    rn2 = block_sums(row_sumsq(a64), row_part)
    qr_, _ = column_basis(at, row_part, rplan.blocks(), dt, rn2)
    mm = at_mul(a64, qc).T @ qr_  # Q_Cᵀ A Q_R
    res2 = a_norm2 - float(np.sum(mm * mm))
    path = "pythagoras"
    if res2 < THETA_EXPLICIT[dt] * a_norm2:
        res2, path = resid_sumsq(a64, qc, qr_ @ mm.T), "explicit"
    u = None
    if want_u:
        c = materialize_columns(a64, col_part, cplan)
        rr = materialize_row_blocks(a64, row_part, rplan)
        tc = qc.T @ c
        tr = qr_.T @ rr.T
        tcp = tc.T @ np.linalg.inv(tc @ tc.T)
        trp = tr.T @ np.linalg.inv(tr @ tr.T)
        u = tcp @ mm @ trp.T
    return CurResult(cplan, rplan, cs, rs, u, math.sqrt(max(res2, 0.0)), math.sqrt(a_norm2), path)


# ----------------------------------------------------------------------------
# Benchmark configurations (BASELINE.json "configs"; unspecified knobs per
# SURVEY Appendix A D11).
# ----------------------------------------------------------------------------

# The single source of the workloads is paper_1703_06065_b200/configs.py (pure data: importing
# it loads no product code).
from paper_1703_06065_b200.configs import CONFIGS  # noqa: E402,F401


# ------------------------------------------------------------------ Algorithm 1
# The reference's default decomposition (blockcur.cpp:54-109): uniform rows → R, approximate
# block leverage of R (leverage.cpp:155-164), g blocks → C = A·S and W = R·S, U = W⁺
# (matcore.cpp:85-91), metrics for U and its rank-k truncation (matcore.cpp:81-83).

@dataclass
class RowDraw:
    row: int
    probability: float
    scale: float


def draw_rows(m: int, r: int, rng: Rng) -> List[RowDraw]:  # sampler.cpp:54-71
    if r < 1 or m < 1:
        raise ValueError("draw_rows: m and r must be >= 1")
    p = 1.0 / m
    scale = 1.0 / math.sqrt(r * p)
    return [RowDraw(rng.below(m), p, scale) for _ in range(r)]


def draw_rows_distinct(m: int, r: int, rng: Rng) -> List[RowDraw]:  # sampler.cpp:73-95
    if r < 1 or m < 1 or r > m:
        raise ValueError("draw_rows_distinct: need 1 <= r <= m")
    pool = list(range(m))
    p = 1.0 / m
    scale = 1.0 / math.sqrt(r * p)
    out = []
    for t in range(r):
        pick = rng.below(m - t)
        pool[t + pick], pool[t] = pool[t], pool[t + pick]
        out.append(RowDraw(pool[t], p, scale))
    return out


def svd_ranked(a: np.ndarray):
    """matcore.cpp:39-56: thin SVD truncated at rank_tolerance."""
    u, s, vt = np.linalg.svd(a, full_matrices=False)
    if s.size == 0:
        return u[:, :0], s[:0], vt[:0]
    tol = rank_tolerance(a.shape[0], a.shape[1], s[0])
    r = int(np.sum((s > tol) & (s > 0)))
    return u[:, :r], s[:r], vt[:r]


def approx_block_leverage(r: np.ndarray, part: BlockPartition) -> ScoreVector:  # leverage.cpp:155-164
    if r.shape[1] != part.n:
        raise DimensionMismatch("approx_block_leverage: partition size does not match R columns")
    if not np.any(r):
        raise ZeroMatrix("approx_block_leverage: R is identically zero")
    _, _, vt = svd_ranked(np.asarray(r, dtype=np.float64))
    return block_leverage(vt.T, part, check=False)


def best_rank_k(a: np.ndarray, k: int) -> np.ndarray:  # matcore.cpp:81-83
    u, s, vt = svd_ranked(np.asarray(a, dtype=np.float64))
    kk = min(k, s.size)
    return (u[:, :kk] * s[:kk]) @ vt[:kk]


@dataclass
class Alg1Result:
    rows: List[RowDraw]
    scores: ScoreVector
    plan: SamplingPlan
    u: np.ndarray
    abs_err_u: float
    abs_err_uk: float
    a_norm: float


def block_cur_alg1(a: np.ndarray, part: BlockPartition, k: int, r: int, g: int, rng: Rng,
                   block_mode: str = WITH_REPLACEMENT, distinct_rows: bool = False) -> Alg1Result:
    """blockcur.cpp:54-109 with row_sampling = uniform (the reference default)."""
    m, n = a.shape
    if k < 1 or k > min(m, n):
        raise ValueError("block_cur: need 1 <= k <= min(m, n)")
    if r < 1 or g < 1:
        raise ValueError("block_cur: r and g must be >= 1")
    if n != part.n:
        raise DimensionMismatch("block_cur: partition does not match A columns")
    a64 = np.asarray(a, dtype=np.float64)
    rows = draw_rows_distinct(m, r, rng) if distinct_rows else draw_rows(m, r, rng)
    rm = np.stack([a64[d.row] * (1.0 if distinct_rows else d.scale) for d in rows])  # materialize_rows
    if not np.any(rm):
        raise DegenerateR("block_cur: sampled row matrix R is identically zero")
    scores = approx_block_leverage(rm, part)
    plan = draw_blocks(scores.distribution(), g, block_mode, rng)
    c = materialize_columns(a64, part, plan)
    w = materialize_columns(rm, part, plan)
    u = pinv(w)
    err_u, _ = error_report(a64, c, u, rm)
    err_uk, _ = error_report(a64, c, best_rank_k(u, k), rm)
    return Alg1Result(rows, scores, plan, u, err_u, err_uk, float(np.linalg.norm(a64)))


def block_cur_alg1_boosted(a, part, k, r, g, t, rng, block_mode=WITH_REPLACEMENT, distinct_rows=False):
    """blockcur.cpp:111-133."""
    best, errors = None, []
    for _ in range(t):
        cur = block_cur_alg1(a, part, k, r, g, rng, block_mode, distinct_rows)
        errors.append(cur.abs_err_u)
        if best is None or cur.abs_err_u < best.abs_err_u:
            best = cur
    return best, errors


# ------------------------------------------------------------------ score diagnostics
def column_block_stable_ranks(m_: np.ndarray, part: BlockPartition) -> np.ndarray:  # leverage.cpp:123-139
    out = np.empty(part.num_blocks())
    for g in range(part.num_blocks()):
        b, e = part.ranges[g]
        slab = np.asarray(m_[:, b:e], dtype=np.float64)
        fro2 = float(np.sum(slab * slab))
        if not fro2 > 0.0:
            raise ZeroBlock(f"column_block_stable_ranks: block {g} has zero Frobenius mass")
        out[g] = fro2 / float(np.linalg.norm(slab, 2)) ** 2
    return out


def block_stable_rank(v_k: np.ndarray, part: BlockPartition) -> float:  # leverage.cpp:141-146
    require_orthonormal(v_k, 1e-8, "block_stable_rank")
    return float(column_block_stable_ranks(np.asarray(v_k).T, part).min())


def incoherence(u_k: np.ndarray) -> float:  # leverage.cpp:148-153
    require_orthonormal(u_k, 1e-8, "incoherence")
    u = np.asarray(u_k, dtype=np.float64)
    return u.shape[0] / u.shape[1] * float(np.max(np.sum(u * u, axis=1)))


# ------------------------------------------------------------------ .bcur files
# io.cpp:105-137 load_matrix_binary and save_matrix_binary (io.hpp:13-14): magic "BCUR",
# little-endian u64 rows, u64 cols, then rows·cols f64 row-major; make_dense's finiteness check
# (matcore.cpp:26-33) surfaces as ParseError.
BCUR_MAGIC = b"BCUR"


def save_matrix_binary(path, a: np.ndarray) -> None:
    a = np.asarray(a, dtype=np.float64)
    with open(path, "wb") as f:
        f.write(BCUR_MAGIC)
        f.write(np.array([a.shape[0], a.shape[1]], dtype="<u8").tobytes())
        f.write(np.ascontiguousarray(a, dtype="<f8").tobytes())


def load_matrix_binary(path) -> np.ndarray:
    try:
        f = open(path, "rb")
    except OSError:
        raise ParseError(f"cannot open {path}")
    with f:
        if f.read(4) != BCUR_MAGIC:
            raise ParseError(f"{path}: missing BCUR magic")
        hdr = f.read(16)
        if len(hdr) != 16:
            raise ParseError(f"{path}: truncated header")
        rows, cols = (int(v) for v in np.frombuffer(hdr, dtype="<u8"))
        if rows == 0 or cols == 0 or rows >= 1 << 31 or cols >= 1 << 31:
            raise ParseError(f"{path}: unreasonable dimensions {rows}x{cols}")
        data = f.read(rows * cols * 8)
        if len(data) != rows * cols * 8:
            raise ParseError(f"{path}: truncated entry data")
    a = np.frombuffer(data, dtype="<f8").reshape(rows, cols).astype(np.float64)
    if not np.all(np.isfinite(a)):
        raise ParseError(f"{path}: matrix contains NaN or Inf")
    return np.asfortranarray(a)


def spectrum(spec: str, r: int) -> np.ndarray:
    kind, *args = spec.split(":")
    i = np.arange(r, dtype=np.float64)
    if kind == "geom":  # σ_i = a·b^i, i = 0..r-1
        return float(args[0]) * float(args[1]) ** i
    if kind == "pow":   # σ_i = i^-e, i = 1..r
        return (i + 1.0) ** (-float(args[0]))
    raise ValueError(spec)
