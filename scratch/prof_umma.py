"""One c3-shaped tcgen05 residual pass (AᵀX with fused row-Σ²) + one sketch pass, for ncu."""
import sys, os, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
from paper_1703_06065_b200 import bcur as B
N = int(os.environ.get("PN", "1024"))
a = B.DeviceMatrix.generate("lowrank", np.float32, 16384, 65536, seed=0, sigma=[1.0] * 8, noise=1e-4)
x = np.asfortranarray(np.random.default_rng(0).standard_normal((16384, N)))
xs = np.asfortranarray(np.random.default_rng(1).standard_normal((65536, 60)))
for _ in range(2):
    B.sketch_product(a, x, transpose=True, row_sumsq=True)
    B.sketch_product(a, xs)
ctx = B.default_context()
ctx.profile(True)
t = time.time()
B.sketch_product(a, x, transpose=True, row_sumsq=True)
B.sketch_product(a, xs)
ctx.synchronize()
print("wall", time.time() - t, ctx.profile_report())
