"""Host-side mirror of the reference's ``bcur::`` hot-path API (proj/include/bcur).

Same names, argument meaning and error behaviour as the reference headers
(leverage.hpp, sampler.hpp, blockcur.hpp, sketch.hpp, matcore.hpp, rng.hpp,
errors.hpp), backed by the sm_100a library through its C ABI
(include/bcur_b200.h).  Matrices are numpy arrays (any order; converted to the
column-major layout of the reference's Eigen ``MatrixXd``) or ``DeviceMatrix``
handles that stay resident in HBM.  fp32 inputs run the fp32 path, everything
else fp64.  There is no CPU compute path: every numeric result comes from the GPU.
"""
from __future__ import annotations

import ctypes as C
import os
import math
from dataclasses import dataclass, field
from typing import List, Optional, Sequence, Tuple

import numpy as np

from . import _lib as L

# --------------------------------------------------------------------------
# errors.hpp:9-57
# --------------------------------------------------------------------------


class Error(RuntimeError):
    """Base of all library failures (errors.hpp:10)."""


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


class DimensionMismatch(Error):
    pass


class ParseError(Error):
    pass


class CudaError(Error):
    """Device failure or no device (the library has no CPU fallback)."""


class CommError(Error):
    pass


_STATUS_EXC = {
    1: ValueError, 2: IndexError, 3: DimensionMismatch, 4: InvalidBasis, 5: ZeroBlock, 6: ZeroMatrix,
    7: DistributionInvalid, 8: NotEnoughBlocks, 9: DegenerateR, 10: IterationFailure, 11: ParseError,
    12: CudaError, 13: CommError,
}


def _check(status: int) -> None:
    if status != L.OK:
        raise _STATUS_EXC.get(status, Error)(L.last_error())


# --------------------------------------------------------------------------
# Device context and matrices
# --------------------------------------------------------------------------


class Context:
    """One GPU, one stream, pooled workspace (bcur_ctx)."""

    def __init__(self, device: int = 0):
        h = C.c_void_p()
        _check(L.lib.bcur_ctx_create(device, C.byref(h)))
        self.handle = h
        self.device = device
        self._comm = None

    def close(self):
        if self.handle:
            L.lib.bcur_ctx_destroy(self.handle)
            self.handle = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def set_stream(self, stream_ptr: Optional[int]):
        _check(L.lib.bcur_ctx_set_stream(self.handle, stream_ptr))

    @property
    def stream(self) -> int:
        return L.lib.bcur_ctx_stream(self.handle) or 0

    def synchronize(self):
        _check(L.lib.bcur_ctx_synchronize(self.handle))

    @property
    def launch_count(self) -> int:
        return int(L.lib.bcur_ctx_launch_count(self.handle))

    def profile(self, enable: bool = True):
        """Start (clear) / stop per-kernel-class CUDA-event accounting."""
        _check(L.lib.bcur_ctx_profile(self.handle, 1 if enable else 0))

    def profile_report(self) -> dict:
        import json
        need = int(L.lib.bcur_ctx_profile_dump(self.handle, None, 0))
        buf = C.create_string_buffer(max(need, 2))
        L.lib.bcur_ctx_profile_dump(self.handle, buf, len(buf))
        return json.loads(buf.value.decode())

    def set_comm(self, rank: int, world: int, allreduce_fn, broadcast_fn=None):
        """allreduce_fn(ptr:int, count:int, stream:int) -> None (in-place sum of fp64);
        broadcast_fn(ptr:int, nbytes:int, root:int, stream:int) -> None (optional)."""
        if world <= 1:
            _check(L.lib.bcur_ctx_set_comm(self.handle, None))
            self._comm = None
            return

        fn = make_comm_callback(allreduce_fn)
        bfn = make_broadcast_callback(broadcast_fn) if broadcast_fn is not None else L.BROADCAST_FN()
        comm = L.CommC(rank, world, None, fn, bfn)
        _check(L.lib.bcur_ctx_set_comm(self.handle, C.byref(comm)))
        self._comm = (fn, bfn, comm)  # keep alive


def make_comm_callback(allreduce_fn):
    """C function pointer for ``bcur_comm.allreduce_f64`` wrapping a Python
    ``allreduce_fn(ptr, count, stream)``; exceptions become a nonzero return, which the
    library reports as BCUR_E_COMM."""
    def cb(user, buf, count, stream):
        try:
            allreduce_fn(C.cast(buf, C.c_void_p).value, int(count), stream or 0)
            return 0
        except Exception:
            import traceback
            traceback.print_exc()
            return 1

    return L.ALLREDUCE_FN(cb)


def make_broadcast_callback(broadcast_fn):
    """C function pointer for ``bcur_comm.broadcast`` wrapping ``broadcast_fn(ptr, nbytes,
    root, stream)``; exceptions become a nonzero return (BCUR_E_COMM)."""
    def cb(user, buf, nbytes, root, stream):
        try:
            broadcast_fn(int(buf or 0), int(nbytes), int(root), stream or 0)
            return 0
        except Exception:
            import traceback
            traceback.print_exc()
            return 1

    return L.BROADCAST_FN(cb)


_default_ctx: Optional[Context] = None


def default_context() -> Context:
    global _default_ctx
    if _default_ctx is None:
        _default_ctx = Context(0)
    return _default_ctx


def _dtype_code(dt) -> int:
    return L.F32 if np.dtype(dt) == np.float32 else L.F64


class DeviceMatrix:
    """Column-major matrix resident in HBM (bcur_dmat)."""

    def __init__(self, handle, ctx: Context, owner=None):
        self.handle = handle
        self.ctx = ctx
        self._owner = owner  # keeps wrapped memory (e.g. a torch tensor) alive
        dt, m, n, ld, p = C.c_int(), L.i64(), L.i64(), L.i64(), C.c_void_p()
        _check(L.lib.bcur_dmat_info(handle, C.byref(dt), C.byref(m), C.byref(n), C.byref(ld), C.byref(p)))
        self.dtype = np.float32 if dt.value == L.F32 else np.float64
        self.shape = (m.value, n.value)
        self.ld = ld.value
        self.ptr = p.value

    @staticmethod
    def from_host(a: np.ndarray, ctx: Optional[Context] = None) -> "DeviceMatrix":
        ctx = ctx or default_context()
        a = np.asarray(a)
        if a.ndim == 1:
            a = a.reshape(-1, 1)
        if a.dtype != np.float32:
            a = a.astype(np.float64, copy=False)
        a = np.asfortranarray(a)
        h = C.c_void_p()
        _check(L.lib.bcur_dmat_create(ctx.handle, _dtype_code(a.dtype), a.shape[0], a.shape[1], C.byref(h)))
        dm = DeviceMatrix(h, ctx)
        _check(L.lib.bcur_dmat_upload(ctx.handle, h, a.ctypes.data_as(C.c_void_p), max(a.shape[0], 1)))
        return dm

    @staticmethod
    def empty(dtype, m: int, n: int, ctx: Optional[Context] = None) -> "DeviceMatrix":
        ctx = ctx or default_context()
        h = C.c_void_p()
        _check(L.lib.bcur_dmat_create(ctx.handle, _dtype_code(np.dtype(dtype)), m, n, C.byref(h)))
        return DeviceMatrix(h, ctx)

    def upload_async(self, host_ptr: int, ld_host: int) -> None:
        """bcur_dmat_upload_async: the copy runs on the context's upload stream; the next call
        that uses this matrix waits for it on the device.  host_ptr (column-major, pinned for an
        asynchronous copy) must stay valid until then."""
        _check(L.lib.bcur_dmat_upload_async(self.ctx.handle, self.handle, C.c_void_p(host_ptr), ld_host))

    @staticmethod
    def load_bcur(path, dtype=np.float64, col0: int = 0, ncols: int = -1,
                  ctx: Optional[Context] = None) -> "DeviceMatrix":
        """io.cpp:105-137 load_matrix_binary, streamed into HBM (column-major, fp32 or fp64);
        columns [col0, col0 + ncols) select a shard.  Raises ParseError like the reference."""
        ctx = ctx or default_context()
        h = C.c_void_p()
        _check(L.lib.bcur_dmat_load_bcur(ctx.handle, os.fsencode(path), _dtype_code(np.dtype(dtype)), col0, ncols,
                                         C.byref(h)))
        return DeviceMatrix(h, ctx)

    def save_bcur(self, path) -> None:
        """save_matrix_binary: row-major fp64 with the BCUR header."""
        _check(L.lib.bcur_dmat_save_bcur(self.ctx.handle, self.handle, os.fsencode(path)))

    @staticmethod
    def wrap(ptr: int, dtype, m: int, n: int, ld: int, ctx: Optional[Context] = None, owner=None) -> "DeviceMatrix":
        ctx = ctx or default_context()
        h = C.c_void_p()
        _check(L.lib.bcur_dmat_wrap(ctx.handle, _dtype_code(dtype), m, n, C.c_void_p(ptr), ld, C.byref(h)))
        return DeviceMatrix(h, ctx, owner)

    @staticmethod
    def generate(kind: str, dtype, m: int, n: int, seed: int, sigma: Sequence[float] = (), noise: float = 0.0,
                 col0: int = 0, n_global: int = 0, ctx: Optional[Context] = None) -> "DeviceMatrix":
        ctx = ctx or default_context()
        sig = np.ascontiguousarray(np.asarray(sigma, dtype=np.float64))
        spec = L.GenSpecC(L.GEN_LOWRANK if kind == "lowrank" else L.GEN_BIOMETRIC, _dtype_code(dtype), m, n,
                          len(sig), sig.ctypes.data_as(L.P_dbl) if len(sig) else None, noise, seed, col0, n_global)
        h = C.c_void_p()
        _check(L.lib.bcur_dmat_generate(ctx.handle, C.byref(spec), C.byref(h)))
        return DeviceMatrix(h, ctx)

    def set_shard(self, col0: int, n_global: int):
        _check(L.lib.bcur_dmat_set_shard(self.handle, col0, n_global))

    def to_host(self) -> np.ndarray:
        out = np.empty(self.shape, dtype=self.dtype, order="F")
        _check(L.lib.bcur_dmat_download(self.ctx.handle, self.handle, out.ctypes.data_as(C.c_void_p),
                                        max(self.shape[0], 1)))
        return out

    def close(self):
        if self.handle:
            L.lib.bcur_dmat_destroy(self.handle)
            self.handle = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def _dev(a, ctx=None) -> DeviceMatrix:
    return a if isinstance(a, DeviceMatrix) else DeviceMatrix.from_host(a, ctx)


# --------------------------------------------------------------------------
# rng.hpp:13-63
# --------------------------------------------------------------------------


class Rng:
    """Seedable generator identical to the reference's (std::mt19937_64 + hand-written draws)."""

    def __init__(self, seed: int):
        h = C.c_void_p()
        _check(L.lib.bcur_rng_create(seed & ((1 << 64) - 1), C.byref(h)))
        self._h = h

    def __del__(self):
        try:
            L.lib.bcur_rng_destroy(self._h)
        except Exception:
            pass

    def seed(self) -> int:
        return int(L.lib.bcur_rng_seed(self._h))

    def next_u64(self) -> int:
        return int(L.lib.bcur_rng_next_u64(self._h))

    def uniform01(self) -> float:
        return float(L.lib.bcur_rng_uniform01(self._h))

    def below(self, bound: int) -> int:
        if bound < 1:
            raise ValueError("below: bound must be >= 1")
        return int(L.lib.bcur_rng_below(self._h, bound))

    def normal(self) -> float:
        return float(L.lib.bcur_rng_normal(self._h))

    def split(self, stream: int) -> "Rng":
        return Rng(int(L.lib.bcur_rng_split_seed(self._h, stream)))

    def uniforms(self, count: int) -> np.ndarray:
        return np.array([self.uniform01() for _ in range(count)], dtype=np.float64)


def omega_key(seed: int) -> int:
    """Sketch key of the pipelines: Rng(seed).split(0x6F6D656761).seed()."""
    return int(L.lib.bcur_omega_key(seed & ((1 << 64) - 1)))


# --------------------------------------------------------------------------
# leverage.hpp:18-82
# --------------------------------------------------------------------------


@dataclass(frozen=True)
class BlockRange:
    begin: int
    end: int

    def width(self) -> int:
        return self.end - self.begin


class BlockPartition:
    """Contiguous disjoint column blocks covering [0, n) (leverage.cpp:27-90)."""

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
        self._n = n
        self._ranges = [BlockRange(int(b), int(e)) for b, e in ranges]
        self._nominal = self.max_width()
        self._off = np.array([r.begin for r in self._ranges] + [n], dtype=np.int64)

    @staticmethod
    def equal_blocks(n: int, block_size: int) -> "BlockPartition":
        if n < 1 or block_size < 1:
            raise ValueError("equal_blocks: n and block_size must be >= 1")
        p = BlockPartition(n, [(b, min(b + block_size, n)) for b in range(0, n, block_size)])
        p._nominal = block_size
        return p

    @staticmethod
    def from_boundaries(n: int, cuts: Sequence[int]) -> "BlockPartition":
        ranges, begin = [], 0
        for c in cuts:
            if c <= begin or c >= n:
                raise ValueError("from_boundaries: cuts must be strictly increasing and inside (0, n)")
            ranges.append((begin, c))
            begin = c
        ranges.append((begin, n))
        return BlockPartition(n, ranges)

    def num_columns(self) -> int:
        return self._n

    def num_blocks(self) -> int:
        return len(self._ranges)

    def range(self, g: int) -> BlockRange:
        if g < 0 or g >= len(self._ranges):
            raise IndexError("BlockPartition::range: block index out of range")
        return self._ranges[g]

    def width(self, g: int) -> int:
        return self.range(g).width()

    def max_width(self) -> int:
        return max(r.width() for r in self._ranges)

    def nominal_block_size(self) -> int:
        return self._nominal

    def ranges(self) -> List[BlockRange]:
        return list(self._ranges)

    def block_of_column(self, j: int) -> int:
        if j < 0 or j >= self._n:
            raise IndexError("block_of_column: column index out of range")
        return int(np.searchsorted(self._off[:-1], j, side="right") - 1)

    def offsets(self) -> np.ndarray:
        return self._off


def _off_ptr(part: BlockPartition):
    off = np.ascontiguousarray(part.offsets(), dtype=np.int64)
    return off, off.ctypes.data_as(L.P_i64)


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


def block_leverage(v_k, part: BlockPartition, tol: float = -1.0, ctx: Optional[Context] = None) -> ScoreVector:
    """Definition-2 block leverage ℓ_g = ‖V_kᵀE_g‖_F² (leverage.cpp:108-121), on the GPU."""
    ctx = ctx or default_context()
    v = _dev(v_k, ctx)
    off, offp = _off_ptr(part)
    G = part.num_blocks()
    out = np.empty(G, dtype=np.float64)
    norm = C.c_double()
    _check(L.lib.bcur_block_leverage(ctx.handle, v.handle, offp, G, tol, out.ctypes.data_as(L.P_dbl), C.byref(norm)))
    return ScoreVector(out, norm.value)


def column_leverage(v_k, tol: float = -1.0, ctx: Optional[Context] = None) -> ScoreVector:
    """Definition-1 column leverage (leverage.cpp:100-106)."""
    ctx = ctx or default_context()
    v = _dev(v_k, ctx)
    out = np.empty(v.shape[0], dtype=np.float64)
    norm = C.c_double()
    _check(L.lib.bcur_column_leverage(ctx.handle, v.handle, tol, out.ctypes.data_as(L.P_dbl), C.byref(norm)))
    return ScoreVector(out, norm.value)


def frobenius_norm(a, ctx: Optional[Context] = None) -> float:  # matcore.cpp:93-95
    ctx = ctx or default_context()
    d = _dev(a, ctx)
    out = C.c_double()
    _check(L.lib.bcur_frobenius_norm(ctx.handle, d.handle, C.byref(out)))
    return out.value


def block_sq_norms(a, part: BlockPartition, ctx: Optional[Context] = None) -> np.ndarray:
    ctx = ctx or default_context()
    d = _dev(a, ctx)
    off, offp = _off_ptr(part)
    out = np.empty(part.num_blocks(), dtype=np.float64)
    _check(L.lib.bcur_block_sq_norms(ctx.handle, d.handle, offp, part.num_blocks(), out.ctypes.data_as(L.P_dbl)))
    return out


def bcur_header(path):
    """(rows, cols) of a .bcur file (plans column shards without reading the data)."""
    r, c = L.i64(), L.i64()
    _check(L.lib.bcur_bcur_header(os.fsencode(path), C.byref(r), C.byref(c)))
    return r.value, c.value


def sketch_product(a, x: np.ndarray, transpose: bool = False, row_sumsq: bool = False,
                   ctx: Optional[Context] = None) -> np.ndarray:
    """A·X (or Aᵀ·X) on the range finder's product kernels; ``row_sumsq`` returns
    Σ_c (AᵀX)_jc² per row without storing the product (fused residual epilogue)."""
    ctx = ctx or default_context()
    d = _dev(a, ctx)
    xd = DeviceMatrix.from_host(np.asarray(x, dtype=np.float64), ctx)
    rows = d.shape[1] if transpose else d.shape[0]
    if row_sumsq:
        out = np.empty(rows, dtype=np.float64)
        _check(L.lib.bcur_sketch_product(ctx.handle, d.handle, xd.handle, 1, None, out.ctypes.data_as(L.P_dbl)))
        return out
    h = C.c_void_p()
    _check(L.lib.bcur_dmat_create(ctx.handle, L.F64, rows, xd.shape[1], C.byref(h)))
    o = DeviceMatrix(h, ctx)
    _check(L.lib.bcur_sketch_product(ctx.handle, d.handle, xd.handle, 1 if transpose else 0, o.handle, None))
    return o.to_host()


def structured_product(a, x: Optional[np.ndarray] = None, transpose: bool = False, gram: bool = False,
                       x_upper: bool = False, rowsq_f16: bool = False, h3: bool = False,
                       fast_acc: bool = False, hi_only: bool = False, ctx: Optional[Context] = None) -> np.ndarray:
    """bcur_sketch_product_ex: ``gram`` → AᵀA (upper triangle valid, ``x`` None);
    ``x_upper`` → A·X or Aᵀ·X with an upper-triangular X (the pipelines' Q = C·R⁻¹);
    ``rowsq_f16`` → Σ_c (AᵀX)_jc² through the pipelines' fp16 row-sum path (n × 1);
    ``h3`` → the same products through the 3×FP16 path (A split into fp16 hi + lo)."""
    ctx = ctx or default_context()
    d = _dev(a, ctx)
    flags = (1 if gram else 0) | (2 if x_upper else 0) | (4 if rowsq_f16 else 0) | (8 if h3 else 0) | \
        (16 if fast_acc else 0) | (32 if hi_only else 0)
    xd = None if x is None else DeviceMatrix.from_host(np.asarray(x, dtype=np.float64), ctx)
    rows = d.shape[1] if (transpose or gram or rowsq_f16) else d.shape[0]
    cols = d.shape[1] if gram else (1 if rowsq_f16 else xd.shape[1])
    h = C.c_void_p()
    _check(L.lib.bcur_dmat_create(ctx.handle, L.F64, rows, cols, C.byref(h)))
    o = DeviceMatrix(h, ctx)
    _check(L.lib.bcur_sketch_product_ex(ctx.handle, d.handle, None if xd is None else xd.handle,
                                        1 if (transpose or gram or rowsq_f16) else 0, flags, o.handle))
    out = o.to_host()
    return out[:, 0] if rowsq_f16 else out


def cholesky(g: np.ndarray, ctx: Optional[Context] = None):
    """G = RᵀR on the device (fp64, upper triangle of g read) → (R, R⁻¹, info, min diag R)."""
    ctx = ctx or default_context()
    g = np.asfortranarray(np.asarray(g, dtype=np.float64))
    w = g.shape[0]
    gd = DeviceMatrix.from_host(g, ctx)
    hs = []
    for _ in range(2):
        h = C.c_void_p()
        _check(L.lib.bcur_dmat_create(ctx.handle, L.F64, w, w, C.byref(h)))
        hs.append(DeviceMatrix(h, ctx))
    info, mn = C.c_int(), C.c_double()
    _check(L.lib.bcur_cholesky(ctx.handle, gd.handle, hs[0].handle, hs[1].handle, C.byref(info), C.byref(mn)))
    return hs[0].to_host(), hs[1].to_host(), info.value, mn.value


@dataclass
class Subspace:
    v_k: np.ndarray
    u_k: np.ndarray
    sigma: np.ndarray
    k_eff: int


def range_finder(a, k: int, p: int, q: int, key: int, ctx: Optional[Context] = None) -> Subspace:
    """Randomized range finder for the top-k right singular subspace (replaces truncate(svd(a),k))."""
    ctx = ctx or default_context()
    d = _dev(a, ctx)
    vh, uh = C.c_void_p(), C.c_void_p()
    sig = np.zeros(k, dtype=np.float64)
    ke = L.i64()
    _check(L.lib.bcur_range_finder(ctx.handle, d.handle, k, p, q, key, C.byref(vh), C.byref(uh),
                                   sig.ctypes.data_as(L.P_dbl), C.byref(ke)))
    v = DeviceMatrix(vh, ctx)
    u = DeviceMatrix(uh, ctx)
    return Subspace(v.to_host(), u.to_host(), sig[:ke.value].copy(), ke.value)


# --------------------------------------------------------------------------
# sampler.hpp:11-72
# --------------------------------------------------------------------------


class SamplingMode:
    with_replacement = "with_replacement"
    without_replacement = "without_replacement"


def _mode_code(mode: str) -> int:
    if mode == SamplingMode.with_replacement:
        return L.WITH_REPLACEMENT
    if mode == SamplingMode.without_replacement:
        return L.WITHOUT_REPLACEMENT
    raise ValueError(f"unknown sampling mode {mode!r}")


@dataclass
class BlockDraw:
    block: int
    probability: float
    scale: float


@dataclass
class SamplingPlan:
    draws: List[BlockDraw] = field(default_factory=list)
    mode: str = SamplingMode.with_replacement
    seed: int = 0
    margins: List[float] = field(default_factory=list)

    def num_draws(self) -> int:
        return len(self.draws)

    def blocks(self) -> List[int]:
        return [d.block for d in self.draws]


def _plan_from_c(arr, n, mode, seed, margins=None) -> SamplingPlan:
    return SamplingPlan([BlockDraw(int(arr[i].block), float(arr[i].probability), float(arr[i].scale))
                         for i in range(n)], mode, seed, list(margins) if margins is not None else [])


def _plan_to_c(plan: SamplingPlan):
    arr = (L.BlockDrawC * max(1, len(plan.draws)))()
    for i, d in enumerate(plan.draws):
        arr[i].block, arr[i].probability, arr[i].scale = d.block, d.probability, d.scale
    return arr


def draw_blocks(probs, g: int, mode: str, rng: Rng, ctx: Optional[Context] = None) -> SamplingPlan:
    """sampler.cpp:116-146 — one uniform per draw from ``rng``; the draw runs on the GPU."""
    ctx = ctx or default_context()
    if g < 1:
        raise ValueError("draw_blocks: g must be >= 1")
    p = np.ascontiguousarray(np.asarray(probs, dtype=np.float64).ravel())
    code = _mode_code(mode)
    u = rng.uniforms(g)
    out = (L.BlockDrawC * g)()
    marg = np.zeros(g, dtype=np.float64)
    _check(L.lib.bcur_draw_blocks(ctx.handle, p.ctypes.data_as(L.P_dbl), p.size, g, code, u.ctypes.data_as(L.P_dbl),
                                  rng.seed(), out, marg.ctypes.data_as(L.P_dbl)))
    return _plan_from_c(out, g, mode, rng.seed(), marg)


def identity_plan(part: BlockPartition) -> SamplingPlan:  # sampler.cpp:148-159
    G = part.num_blocks()
    return SamplingPlan([BlockDraw(j, 1.0 / G, 1.0) for j in range(G)], SamplingMode.without_replacement, 0)


def materialize_columns(a, part: BlockPartition, plan: SamplingPlan, ctx: Optional[Context] = None,
                        on_device: bool = False):
    """C = A S (sampler.cpp:161-184), gathered on the GPU."""
    ctx = ctx or default_context()
    d = _dev(a, ctx)
    off, offp = _off_ptr(part)
    arr = _plan_to_c(plan)
    h = C.c_void_p()
    _check(L.lib.bcur_materialize_columns(ctx.handle, d.handle, offp, part.num_blocks(), arr, len(plan.draws),
                                          C.byref(h)))
    out = DeviceMatrix(h, ctx)
    return out if on_device else out.to_host()


def materialize_row_blocks(a, part: BlockPartition, plan: SamplingPlan, ctx: Optional[Context] = None,
                           on_device: bool = False):
    """R = S_Rᵀ A for row blocks (row blocks = column blocks of Aᵀ)."""
    ctx = ctx or default_context()
    d = _dev(a, ctx)
    off, offp = _off_ptr(part)
    arr = _plan_to_c(plan)
    h = C.c_void_p()
    _check(L.lib.bcur_materialize_row_blocks(ctx.handle, d.handle, offp, part.num_blocks(), arr, len(plan.draws),
                                             C.byref(h)))
    out = DeviceMatrix(h, ctx)
    return out if on_device else out.to_host()


# --------------------------------------------------------------------------
# blockcur.hpp / sketch.hpp
# --------------------------------------------------------------------------


@dataclass
class ErrorReport:
    abs_err: float
    rel_to_a: float
    rel_to_best_k: Optional[float] = None
    k: int = 0
    variant: str = "U"


@dataclass
class ErrorBaseline:
    a_norm: float
    best_k_residual: float
    k: int


def error_report(a, c, u, r, k: int = 0, variant: str = "U", baseline: Optional[ErrorBaseline] = None,
                 ctx: Optional[Context] = None) -> ErrorReport:
    """blockcur.cpp:33-52: ‖A − C(UR)‖_F on the GPU.  ``rel_to_best_k`` needs a baseline
    (the reference computes it from a full SVD of A, which this path does not run)."""
    ctx = ctx or default_context()
    da, dc, du, dr = (_dev(x, ctx) for x in (a, c, u, r))
    ae, an = C.c_double(), C.c_double()
    _check(L.lib.bcur_error_report(ctx.handle, da.handle, dc.handle, du.handle, dr.handle, C.byref(ae), C.byref(an)))
    rel = ae.value / an.value if an.value > 0 else 0.0
    rbk = None
    if baseline is not None and baseline.best_k_residual >= 1e-12:
        rbk = ae.value / baseline.best_k_residual
    return ErrorReport(ae.value, rel, rbk, k, variant)


@dataclass
class CssResult:
    """sketch.hpp:32-36 (+ scores, report and per-draw margins)."""
    c: Optional[np.ndarray]
    projection_error: float
    plan: SamplingPlan
    scores: ScoreVector
    a_norm: float
    rank_c: int
    residual_path: str
    orth_dev: float

    @property
    def rel_err(self) -> float:
        return self.projection_error / self.a_norm if self.a_norm > 0 else 0.0


def _options(k, p, q, g, g_rows, mode, residual, seed, rank_floor=False):
    return L.OptionsC(k, p, q, g, g_rows, _mode_code(mode), residual, seed & ((1 << 64) - 1), int(bool(rank_floor)))


def block_css(a, part: BlockPartition, k: int, g: int, rng: Rng, p: int = 5, q: int = 0,
              mode: str = SamplingMode.with_replacement, residual: int = L.RESID_AUTO, return_c: bool = True,
              ctx: Optional[Context] = None, rank_floor: bool = False) -> CssResult:
    """Block column subset selection (sketch.cpp:68-82): block leverage at rank k from the
    randomized range finder (sketch key from ``rng.seed()``), g draws (one uniform each
    from ``rng``), C = A S, projection error ‖A − CC⁺A‖_F — all on the GPU."""
    ctx = ctx or default_context()
    if k < 1:
        raise ValueError("block_css: k must be >= 1")
    if g < 1:
        raise ValueError("draw_blocks: g must be >= 1")
    d = _dev(a, ctx)
    off, offp = _off_ptr(part)
    G = part.num_blocks()
    u = rng.uniforms(g)
    opt = _options(k, p, q, g, 0, mode, residual, rng.seed(), rank_floor)
    scores = np.empty(G, dtype=np.float64)
    norm = C.c_double()
    draws = (L.BlockDrawC * g)()
    marg = np.zeros(g, dtype=np.float64)
    rep = L.ReportC()
    _check(L.lib.bcur_block_css(ctx.handle, d.handle, offp, G, C.byref(opt), u.ctypes.data_as(L.P_dbl),
                                scores.ctypes.data_as(L.P_dbl), C.byref(norm), draws, marg.ctypes.data_as(L.P_dbl),
                                C.byref(rep)))
    plan = _plan_from_c(draws, g, mode, rng.seed(), marg)
    cm = materialize_columns(d, part, plan, ctx) if return_c else None
    return CssResult(cm, rep.abs_err, plan, ScoreVector(scores, norm.value), rep.a_norm, rep.rank_c,
                     "explicit" if rep.residual_path else "pythagoras", rep.orth_dev)


def block_diagnostics(v_k, u_k, part: BlockPartition, ctx: Optional[Context] = None):
    """leverage.cpp:123-153 on the GPU: (per-block stable ranks of V_kᵀ, their minimum =
    block_stable_rank, incoherence of U_k).  A zero-mass block raises ZeroBlock like the
    reference (``bcur scores`` then reports NaN)."""
    ctx = ctx or default_context()
    dv = _dev(v_k, ctx)
    du = _dev(u_k, ctx) if u_k is not None else None
    off, offp = _off_ptr(part)
    G = part.num_blocks()
    sr = np.empty(G, dtype=np.float64)
    alpha, mu = C.c_double(), C.c_double()
    _check(L.lib.bcur_block_diagnostics(ctx.handle, dv.handle, du.handle if du is not None else None, offp, G,
                                        sr.ctypes.data_as(L.P_dbl), C.byref(alpha), C.byref(mu)))
    return sr, alpha.value, (mu.value if du is not None else float("nan"))


# -------------------------------------------- Algorithm 1 (blockcur.cpp:54-109)
@dataclass
class RowDraw:
    row: int
    probability: float
    scale: float


def draw_rows(m: int, r: int, rng: Rng) -> List[RowDraw]:
    """sampler.cpp:54-71: r uniform draws with replacement, one ``rng.below(m)`` each."""
    if r < 1 or m < 1:
        raise ValueError("draw_rows: m and r must be >= 1")
    p = 1.0 / m
    scale = 1.0 / math.sqrt(r * p)
    return [RowDraw(rng.below(m), p, scale) for _ in range(r)]


def draw_rows_distinct(m: int, r: int, rng: Rng) -> List[RowDraw]:
    """sampler.cpp:73-95: partial Fisher–Yates over 0..m-1."""
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


@dataclass
class CurResultAlg1:
    rows: List[RowDraw]
    scores: ScoreVector
    block_plan: SamplingPlan
    u: np.ndarray
    abs_err_u: float
    abs_err_uk: float
    a_norm: float
    rank_w: int

    @property
    def rel_to_a(self) -> float:
        return self.abs_err_u / self.a_norm if self.a_norm > 0 else 0.0


def block_cur_reference(a, part: BlockPartition, k: int, r: int, g: int, rng: Rng,
                        block_mode: str = SamplingMode.with_replacement, distinct_rows: bool = False,
                        ctx: Optional[Context] = None) -> CurResultAlg1:
    """The reference's default block CUR (blockcur.cpp:54-109, row_sampling = uniform): the
    rows are drawn here from ``rng`` exactly as draw_rows / draw_rows_distinct, then one
    uniform per block draw; everything else (approximate block leverage of R, C, W,
    U = W⁺, both error metrics) runs on the GPU."""
    ctx = ctx or default_context()
    d = _dev(a, ctx)
    m = d.shape[0]
    if k < 1 or k > min(d.shape):
        raise ValueError("block_cur: need 1 <= k <= min(m, n)")
    if r < 1 or g < 1:
        raise ValueError("block_cur: r and g must be >= 1")
    rows = draw_rows_distinct(m, r, rng) if distinct_rows else draw_rows(m, r, rng)
    rc = (L.RowDrawC * r)(*[L.RowDrawC(x.row, x.probability, x.scale) for x in rows])
    u = rng.uniforms(g)
    off, offp = _off_ptr(part)
    G = part.num_blocks()
    scores = np.empty(G, dtype=np.float64)
    norm = C.c_double()
    draws = (L.BlockDrawC * g)()
    marg = np.zeros(g, dtype=np.float64)
    rep = L.Alg1ReportC()
    # U is c × r with c = the drawn blocks' total width (≤ the g widest blocks); the library
    # writes it contiguously (ld = c) at the start of this buffer
    cap = sum(sorted((part.width(b) for b in range(G)), reverse=True)[:g]) * r
    ubuf = np.empty(max(cap, 1), dtype=np.float64)
    _check(L.lib.bcur_block_cur_alg1(ctx.handle, d.handle, offp, G, k, rc, r, 0 if distinct_rows else 1, g,
                                     _mode_code(block_mode), u.ctypes.data_as(L.P_dbl), scores.ctypes.data_as(L.P_dbl),
                                     C.byref(norm), draws, marg.ctypes.data_as(L.P_dbl), ubuf.ctypes.data_as(L.P_dbl),
                                     C.byref(rep)))
    plan = _plan_from_c(draws, g, block_mode, rng.seed(), marg)
    cc = sum(part.width(dr.block) for dr in plan.draws)
    um = ubuf[:cc * r].reshape((cc, r), order="F").copy(order="F")
    return CurResultAlg1(rows, ScoreVector(scores, norm.value), plan, um, rep.abs_err_u, rep.abs_err_uk, rep.a_norm,
                         rep.rank_w)


def block_cur_reference_boosted(a, part: BlockPartition, k: int, r: int, g: int, t: int, rng: Rng,
                                block_mode: str = SamplingMode.with_replacement, distinct_rows: bool = False,
                                ctx: Optional[Context] = None):
    """blockcur.cpp:111-133: t trials on one Rng stream, the lowest ‖A − CUR‖_F kept;
    returns (best, [abs_err of every trial])."""
    if t < 1:
        raise ValueError("block_cur_boosted: t must be >= 1")
    ctx = ctx or default_context()
    d = _dev(a, ctx)
    best, errors = None, []
    for _ in range(t):
        cur = block_cur_reference(d, part, k, r, g, rng, block_mode, distinct_rows, ctx)
        errors.append(cur.abs_err_u)
        if best is None or cur.abs_err_u < best.abs_err_u:
            best = cur
    return best, errors


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


def greedy_select(a, part: BlockPartition, k: int, g: int, seed: int, p: int = 5, q: int = 0,
                  residual: int = L.RESID_AUTO, ctx: Optional[Context] = None) -> GreedyResult:
    """Greedy deterministic block selection by residual mass ‖(I−P_C)A_g‖_F²."""
    ctx = ctx or default_context()
    d = _dev(a, ctx)
    off, offp = _off_ptr(part)
    G = part.num_blocks()
    opt = _options(k, p, q, g, 0, SamplingMode.without_replacement, residual, seed)
    steps = (L.GreedyStepC * max(g, 1))()
    res = np.empty(G, dtype=np.float64)
    rep = L.ReportC()
    _check(L.lib.bcur_greedy_select(ctx.handle, d.handle, offp, G, C.byref(opt), steps, res.ctypes.data_as(L.P_dbl),
                                    C.byref(rep)))
    st = [GreedyStep(int(steps[i].block), float(steps[i].score), float(steps[i].margin), bool(steps[i].saturated),
                     int(steps[i].rank_added)) for i in range(g)]
    return GreedyResult(st, rep.abs_err, rep.a_norm, res, "explicit" if rep.residual_path else "pythagoras")


@dataclass
class CurResult:
    col_plan: SamplingPlan
    row_plan: SamplingPlan
    col_scores: ScoreVector
    row_scores: ScoreVector
    u: Optional[np.ndarray]
    abs_err: float
    a_norm: float
    rank_c: int
    rank_r: int
    residual_path: str

    @property
    def rel_err(self) -> float:
        return self.abs_err / self.a_norm if self.a_norm > 0 else 0.0


def pinned_empty(shape, dtype=np.float64, order: str = "F") -> np.ndarray:
    """An uninitialized array in page-locked host memory (bcur_host_alloc): as an upload source it
    makes the copy asynchronous, as a result buffer (``block_cur(..., out_u=...)``) it takes one DMA
    copy where pageable memory is staged.  Freed with the array."""
    import weakref

    shape = (shape,) if np.isscalar(shape) else tuple(int(x) for x in shape)
    dt = np.dtype(dtype)
    nbytes = int(np.prod(shape, dtype=np.int64)) * dt.itemsize
    ptr = C.c_void_p()
    _check(L.lib.bcur_host_alloc(max(nbytes, 1), C.byref(ptr)))
    buf = (C.c_char * max(nbytes, 1)).from_address(ptr.value)
    arr = np.frombuffer(buf, dtype=dt, count=int(np.prod(shape, dtype=np.int64))).reshape(shape, order=order)
    weakref.finalize(buf, L.lib.bcur_host_free, ptr)  # buf lives as long as any view of it
    return arr


def block_cur(a, col_part: BlockPartition, row_part: BlockPartition, k: int, gc: int, gr: int, rng: Rng,
              p: int = 10, q: int = 0, mode: str = SamplingMode.without_replacement, want_u: bool = True,
              residual: int = L.RESID_AUTO, ctx: Optional[Context] = None, rank_floor: bool = False,
              out_u: Optional[np.ndarray] = None) -> CurResult:
    """Block CUR with row and column blocks: U = C⁺AR⁺ and ‖A − CUR‖_F on the GPU.

    ``out_u``: a caller-owned Fortran-ordered float64 buffer of at least (gc·max col width) ×
    (gr·max row width) that receives U (the result's ``u`` is a view of it) — a serving loop
    reuses one ``pinned_empty`` buffer, which takes U in one DMA copy."""
    ctx = ctx or default_context()
    d = _dev(a, ctx)
    coff, coffp = _off_ptr(col_part)
    roff, roffp = _off_ptr(row_part)
    Gc, Gr = col_part.num_blocks(), row_part.num_blocks()
    u = rng.uniforms(gc + gr)
    opt = _options(k, p, q, gc, gr, mode, residual, rng.seed(), rank_floor)
    cs = np.empty(Gc)
    rs = np.empty(Gr)
    cd = (L.BlockDrawC * gc)()
    rd = (L.BlockDrawC * gr)()
    rep = L.ReportC()
    umat = None
    if want_u:
        # upper bound on the factor sizes: every draw takes the widest block
        cmax = gc * col_part.max_width()
        rmax = gr * row_part.max_width()
        if out_u is not None:
            if (out_u.dtype != np.float64 or out_u.ndim != 2 or not out_u.flags.f_contiguous
                    or out_u.shape[0] < cmax or out_u.shape[1] < rmax):
                raise ValueError("block_cur: out_u must be Fortran-ordered float64 of at least %d x %d" % (cmax, rmax))
            umat = out_u
        else:
            umat = np.empty((cmax, rmax), dtype=np.float64, order="F")  # only [:cw, :rw] is returned
    _check(L.lib.bcur_block_cur(ctx.handle, d.handle, coffp, Gc, roffp, Gr, C.byref(opt), u.ctypes.data_as(L.P_dbl),
                                cs.ctypes.data_as(L.P_dbl), rs.ctypes.data_as(L.P_dbl), cd, rd,
                                umat.ctypes.data_as(L.P_dbl) if want_u else None, umat.shape[0] if want_u else 1,
                                C.byref(rep)))
    cplan = _plan_from_c(cd, gc, mode, rng.seed())
    rplan = _plan_from_c(rd, gr, mode, rng.seed())
    if want_u:
        cw = sum(col_part.width(x.block) for x in cplan.draws)
        rw = sum(row_part.width(x.block) for x in rplan.draws)
        umat = umat[:cw, :rw] if out_u is not None else np.asfortranarray(umat[:cw, :rw])
    return CurResult(cplan, rplan, ScoreVector(cs, float(rep.k_eff)), ScoreVector(rs, float(rep.k_eff)), umat,
                     rep.abs_err, rep.a_norm, rep.rank_c, rep.rank_r,
                     "explicit" if rep.residual_path else "pythagoras")


def boost_trials(delta: float) -> int:  # blockcur.cpp:146-151
    if not (0.0 < delta < 1.0):
        raise ValueError("boost_trials: delta must be in (0, 1)")
    return int(math.ceil(math.log(1.0 / delta)))
