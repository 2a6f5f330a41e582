"""c3-shaped range-finder passes (A·X, Aᵀ·Q, N = 60) under BCUR_UMMA_DEBUG role switches:
prints the per-pass ms so the limiting role shows (results are wrong with switches on)."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
from paper_1703_06065_b200 import bcur as B
a = B.DeviceMatrix.generate("lowrank", np.float32, 16384, 65536, seed=0, sigma=[1.0] * 8, noise=1e-4)
xs = np.asfortranarray(np.random.default_rng(1).standard_normal((65536, 60)))
q60 = np.asfortranarray(np.random.default_rng(2).standard_normal((16384, 60)))
ctx = B.default_context()
for it in range(3):
    if it == 2:
        ctx.profile(True)
    B.sketch_product(a, xs)
    B.sketch_product(a, q60, transpose=True)
rep = ctx.profile_report()
print("dbg", os.environ.get("BCUR_UMMA_DEBUG", "0"), {k: round(v["ms"] / max(v["scopes"], 1), 3) for k, v in rep.items() if k.startswith("umma")})
