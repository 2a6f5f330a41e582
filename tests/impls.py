"""Run the reference's ported tests against both implementations of the path:
the CPU oracle (checker) and the GPU product (through its C ABI)."""
import numpy as np
import pytest

from oracle import bcur_oracle as O


class OracleImpl:
    name = "oracle"
    Rng = O.Rng
    BlockPartition = O.BlockPartition
    InvalidBasis = O.InvalidBasis
    DistributionInvalid = O.DistributionInvalid
    NotEnoughBlocks = O.NotEnoughBlocks
    DimensionMismatch = O.DimensionMismatch
    ZeroMatrix = O.ZeroMatrix
    WITH = O.WITH_REPLACEMENT
    WITHOUT = O.WITHOUT_REPLACEMENT

    @staticmethod
    def block_leverage(v, part):
        tol = O.ORTHONORMAL_TOL.get(np.dtype(v.dtype), 1e-8)
        return O.block_leverage(v, part, tol)

    @staticmethod
    def column_leverage(v):
        return O.column_leverage(v)

    @staticmethod
    def draw_blocks(probs, g, mode, rng):
        return O.draw_blocks(np.asarray(probs, dtype=np.float64), g, mode, rng)

    @staticmethod
    def materialize_columns(a, part, blocks_scales):
        plan = O.SamplingPlan([O.BlockDraw(b, p, s) for b, p, s in blocks_scales])
        return O.materialize_columns(np.asarray(a), part, plan)

    @staticmethod
    def identity_plan(part):
        return [(d.block, d.probability, d.scale) for d in O.identity_plan(part).draws]

    @staticmethod
    def block_css(a, part, k, g, rng, p=5, q=0, mode=O.WITH_REPLACEMENT):
        r = O.block_css(np.asarray(a), part, k, g, rng, p=p, q=q, mode=mode)
        return r.plan.blocks(), r.abs_err, r.scores.scores

    @staticmethod
    def error_report(a, c, u, r):
        return O.error_report(a, c, u, r)


class GpuImpl:
    name = "gpu"

    def __init__(self):
        from paper_1703_06065_b200 import bcur as B
        self.B = B
        self.Rng = B.Rng
        self.BlockPartition = B.BlockPartition
        self.InvalidBasis = B.InvalidBasis
        self.DistributionInvalid = B.DistributionInvalid
        self.NotEnoughBlocks = B.NotEnoughBlocks
        self.DimensionMismatch = B.DimensionMismatch
        self.ZeroMatrix = B.ZeroMatrix
        self.WITH = B.SamplingMode.with_replacement
        self.WITHOUT = B.SamplingMode.without_replacement

    def block_leverage(self, v, part):
        return self.B.block_leverage(v, part)

    def column_leverage(self, v):
        return self.B.column_leverage(v)

    def draw_blocks(self, probs, g, mode, rng):
        return self.B.draw_blocks(probs, g, mode, rng)

    def materialize_columns(self, a, part, blocks_scales):
        plan = self.B.SamplingPlan([self.B.BlockDraw(b, p, s) for b, p, s in blocks_scales])
        return self.B.materialize_columns(a, part, plan)

    def identity_plan(self, part):
        return [(d.block, d.probability, d.scale) for d in self.B.identity_plan(part).draws]

    def block_css(self, a, part, k, g, rng, p=5, q=0, mode=None):
        mode = mode or self.WITH
        r = self.B.block_css(a, part, k, g, rng, p=p, q=q, mode=mode, return_c=False)
        return r.plan.blocks(), r.projection_error, r.scores.scores

    def error_report(self, a, c, u, r):
        rep = self.B.error_report(a, c, u, r)
        return rep.abs_err, rep.rel_to_a


@pytest.fixture(params=["oracle", pytest.param("gpu", marks=pytest.mark.gpu)])
def impl(request):
    if request.param == "oracle":
        return OracleImpl()
    return GpuImpl()
