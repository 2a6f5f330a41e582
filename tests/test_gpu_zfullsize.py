"""Full-size parity of the BASELINE.json configs against the CPU oracle (north star:
"oracle-matching block selections and CUR error on all five configs").

A is generated on the device (Philox; the same generator the bench times), copied to
the host as stored (fp32), and the oracle runs on exactly those values in fp64
(column-chunked, oracle/bcur_oracle.py a_mul/at_mul).  Bars: identical selections except
after a recorded near-tie (D14), block scores within 1e-4 relative (fp32), reconstruction
error within 1e-6 relative.

  c3  16384 × 65536 fp32, k=50 p=10 q=2, 32 of 512 blocks — the bench headline; its residual
      takes the Pythagoras path (rel_err ≈ 0.80) through the fp16 row-Σ² pass.
  c4  32768² fp32, 24 row + 24 column blocks, U = C⁺AR⁺.
  c5  65536 × 262144 fp32 (68.7 GB on one GPU): the leverage part — block scores of the
      rank-200 subspace and the 64 draws (the oracle's fp64 QᵀA of the residual, 2.8e14 flop,
      does not fit a test's CPU budget).

The c3 result is also written to gpurun_out/golden_c3.json (checksums of A, plan, scores,
error); the committed copy is tests/golden/c3.json, checked without the oracle by
test_golden.py.  The file name sorts last so the quick tests run first under -x.
"""
import json
import os
import struct
import time

import numpy as np
import pytest

from oracle import bcur_oracle as O
from paper_1703_06065_b200.configs import CONFIGS, spectrum

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def hexd(x):
    return struct.pack(">d", float(x)).hex()


def gen(B, name):
    c = CONFIGS[name]
    dt = np.float32 if c["dtype"] == "f32" else np.float64
    return B.DeviceMatrix.generate("lowrank", dt, c["m"], c["n"], seed=c["seed"],
                                   sigma=spectrum(c["spectrum"], c["rank"]), noise=c["noise"])


def rel_max(got, ref):
    got, ref = np.asarray(got, dtype=np.float64), np.asarray(ref, dtype=np.float64)
    return float(np.max(np.abs(got - ref) / np.maximum(np.abs(ref), 1e-300)))


def plans_agree(got, ref_plan):
    """Identical draws up to the first recorded near-tie (D14)."""
    for t, (bg, dr) in enumerate(zip(got, ref_plan.draws)):
        if ref_plan.margins[t] < 1e-9:
            return t
        assert bg == dr.block, (t, got, ref_plan.blocks())
    return len(got)


def checksums(a):
    s, s2 = 0.0, 0.0
    for j0, j1 in O._chunks(a):
        c = O.cols64(a, j0, j1)
        s += float(np.sum(c))
        s2 += float(np.einsum("ij,ij->", c, c))
    return {"sum": hexd(s), "sumsq": hexd(s2), "corner": [hexd(a[0, 0]), hexd(a[-1, -1])]}


def test_c3_full_size_matches_oracle():
    from paper_1703_06065_b200 import bcur as B
    c = CONFIGS["c3"]
    dm = gen(B, "c3")
    part = B.BlockPartition.equal_blocks(c["n"], c["s"])
    got = B.block_css(dm, part, c["k"], c["g"], B.Rng(c["seed"]), p=c["p"], q=c["q"], mode=c["mode"],
                      return_c=False)
    a = dm.to_host()
    dm.close()
    t0 = time.time()
    ref = O.block_css(a, O.BlockPartition.equal_blocks(c["n"], c["s"]), c["k"], c["g"], O.Rng(c["seed"]),
                      p=c["p"], q=c["q"], mode=c["mode"])
    oracle_s = time.time() - t0
    score_rel = rel_max(got.scores.scores, ref.scores.scores)
    err_rel = abs(got.projection_error - ref.abs_err) / ref.abs_err
    out = {"config": "c3", "dtype": "float32", "m": c["m"], "n": c["n"], "s": c["s"], "k": c["k"], "p": c["p"],
           "q": c["q"], "g": c["g"], "mode": c["mode"], "seed": c["seed"], "rank": c["rank"],
           "spectrum": c["spectrum"], "noise": c["noise"], "a": checksums(a),
           "scores": [hexd(x) for x in ref.scores.scores], "normalizer": ref.scores.normalizer,
           "plan": {"blocks": ref.plan.blocks(), "margins": [float(x) for x in ref.plan.margins]},
           "abs_err": hexd(ref.abs_err), "a_norm": hexd(ref.a_norm), "rank_c": ref.rank_c,
           "residual_path": ref.residual_path,
           "gpu": {"blocks": got.plan.blocks(), "abs_err": got.projection_error, "score_rel_max": score_rel,
                   "err_rel": err_rel, "residual_path": got.residual_path},
           "oracle_seconds": oracle_s}
    os.makedirs(os.path.join(ROOT, "gpurun_out"), exist_ok=True)
    with open(os.path.join(ROOT, "gpurun_out", "golden_c3.json"), "w") as f:
        json.dump(out, f, indent=1)
    assert ref.residual_path == "pythagoras" and got.residual_path == "pythagoras"
    assert score_rel <= 1e-4, score_rel
    assert got.scores.normalizer == ref.scores.normalizer
    assert plans_agree(got.plan.blocks(), ref.plan) == c["g"]
    assert got.rank_c == ref.rank_c
    assert err_rel <= 1e-6, (got.projection_error, ref.abs_err)
    assert got.a_norm == pytest.approx(ref.a_norm, rel=1e-10)


def test_c4_full_size_matches_oracle():
    from paper_1703_06065_b200 import bcur as B
    c = CONFIGS["c4"]
    dm = gen(B, "c4")
    cg, rg = B.BlockPartition.equal_blocks(c["n"], c["s"]), B.BlockPartition.equal_blocks(c["m"], c["s"])
    got = B.block_cur(dm, cg, rg, c["k"], c["g"], c["g_rows"], B.Rng(c["seed"]), p=c["p"], q=c["q"],
                      mode=c["mode"], want_u=True)
    a = dm.to_host()
    dm.close()
    co, ro = O.BlockPartition.equal_blocks(c["n"], c["s"]), O.BlockPartition.equal_blocks(c["m"], c["s"])
    ref = O.block_cur_rows_cols(a, co, ro, c["k"], c["g"], c["g_rows"], O.Rng(c["seed"]), p=c["p"], q=c["q"],
                                mode=c["mode"], want_u=True)
    assert rel_max(got.col_scores.scores, ref.col_scores.scores) <= 1e-4
    assert rel_max(got.row_scores.scores, ref.row_scores.scores) <= 1e-4
    assert plans_agree(got.col_plan.blocks(), ref.col_plan) == c["g"]
    assert plans_agree(got.row_plan.blocks(), ref.row_plan) == c["g_rows"]
    assert abs(got.abs_err - ref.abs_err) <= 1e-6 * ref.abs_err, (got.abs_err, ref.abs_err)
    assert got.u.shape == ref.u.shape
    assert np.max(np.abs(got.u - ref.u)) <= 1e-4 * np.max(np.abs(ref.u))


def test_c5_full_size_leverage_matches_oracle():
    from paper_1703_06065_b200 import bcur as B
    c = CONFIGS["c5"]
    dm = gen(B, "c5")
    part = B.BlockPartition.equal_blocks(c["n"], c["s"])
    got = B.block_css(dm, part, c["k"], c["g"], B.Rng(c["seed"]), p=c["p"], q=c["q"], mode=c["mode"],
                      return_c=False)
    a = dm.to_host()
    dm.close()
    sub = O.range_finder(a, c["k"], c["p"], c["q"], O.omega_key_from_seed(c["seed"]))
    del a
    po = O.BlockPartition.equal_blocks(c["n"], c["s"])
    scores = O.block_leverage(sub.v_k, po, check=False)
    plan = O.draw_blocks(scores.distribution(), c["g"], c["mode"], O.Rng(c["seed"]))
    assert got.scores.normalizer == scores.normalizer == sub.k_eff
    assert rel_max(got.scores.scores, scores.scores) <= 1e-4
    assert plans_agree(got.plan.blocks(), plan) == c["g"]
