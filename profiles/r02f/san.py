"""Small decompositions for compute-sanitizer (memcheck / racecheck / synccheck): c1 (fp64, DMMA,
Cholesky leaves), a small fp32 css (tcgen05 3×FP16 range finder, CTA-pair row-Σ², whole-C CholQR2
with the recursive factorization), greedy and CUR."""
import sys, os
sys.path.insert(0, os.environ.get("GRAFT_REPO_ROOT", "/root/repo"))
import numpy as np
from oracle import bcur_oracle as O
from paper_1703_06065_b200 import bcur as B
c = O.CONFIGS["c1"]
a = O.gen_lowrank(c["m"], c["n"], O.spectrum(c["spectrum"], c["rank"]), c["noise"], c["seed"])
r = B.block_css(a, B.BlockPartition.equal_blocks(c["n"], c["s"]), c["k"], c["g"], B.Rng(0), p=c["p"], q=c["q"], mode=c["mode"])
print("c1", r.plan.blocks(), r.rel_err)
a = O.gen_lowrank(1024, 4096, 30, "pow:1", 1e-4, 3, dtype=np.float32)
part = B.BlockPartition.equal_blocks(4096, 128)
r = B.block_css(a, part, 20, 6, B.Rng(1), p=10, q=1, mode=B.SamplingMode.without_replacement, return_c=False)
print("css f32", r.plan.blocks(), r.rel_err, r.residual_path)
r = B.block_css(a, part, 20, 6, B.Rng(1), p=10, q=1, mode=B.SamplingMode.without_replacement, return_c=False, residual=B.L.RESID_EXPLICIT)
print("css f32 explicit", r.rel_err)
g = B.greedy_select(a, part, 20, 4, seed=2, p=10)
print("greedy", g.blocks(), g.rel_err)
cu = B.block_cur(a, part, B.BlockPartition.equal_blocks(1024, 128), 20, 3, 2, B.Rng(3), p=10)
print("cur", cu.rel_err)
