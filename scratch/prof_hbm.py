"""HBM-bound tcgen05 passes at c3 size for ncu: sketch AX (N=60), AtX store (N=60), greedy rowsq (N=128)."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
from paper_1703_06065_b200 import bcur as B
a = B.DeviceMatrix.generate("lowrank", np.float32, 16384, 65536, seed=0, sigma=[1.0] * 8, noise=1e-4)
xs = np.asfortranarray(np.random.default_rng(1).standard_normal((65536, 60)))
q60 = np.asfortranarray(np.random.default_rng(2).standard_normal((16384, 60)))
q128 = np.asfortranarray(np.random.default_rng(3).standard_normal((16384, 128)))
for it in range(3):
    if it == 2:
        ctx = B.default_context(); ctx.profile(True)
    B.sketch_product(a, xs)
    B.sketch_product(a, q60, transpose=True)
    B.sketch_product(a, q128, transpose=True, row_sumsq=True)
print(B.default_context().profile_report())
