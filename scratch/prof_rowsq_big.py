"""c3-shaped row-Σ² on a pre-rounded A (the path block_css takes): 16384×65536 A, N=4096 basis."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
from paper_1703_06065_b200 import bcur as B
N = int(os.environ.get("PN", "4096"))
a = B.DeviceMatrix.generate("lowrank", np.float32, 16384, 65536, seed=0, sigma=[1.0] * 8, noise=1e-4)
part = B.BlockPartition.equal_blocks(65536, 128)
ctx = B.default_context()
# one warm and one profiled block_css with g = N/128 blocks (the residual is the X1 pass)
for it in range(2):
    if it == 1:
        ctx.profile(True)
    r = B.block_css(a, part, 50, N // 128, B.Rng(0), p=10, q=0, mode="without_replacement", return_c=False)
rep = ctx.profile_report()
print({k: round(v["ms"], 3) for k, v in rep.items() if k in ("umma_atx_rowsq", "phase:5 residual")}, r.rel_err)
