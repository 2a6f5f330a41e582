"""c3 basis-shaped compute-bound tcgen05 passes for ncu: Gram CᵀC (16384×4096) and C·R⁻¹ (4096²)."""
import sys, os, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
from paper_1703_06065_b200 import bcur as B
m, w = 16384, 4096
a = B.DeviceMatrix.generate("lowrank", np.float32, m, w, seed=0, sigma=[1.0] * 8, noise=1e-2)
x = np.asfortranarray(np.random.default_rng(0).standard_normal((m, w)))
r = np.asfortranarray(np.triu(np.random.default_rng(1).standard_normal((w, w))))
for it in range(2):
    if it == 1:
        ctx = B.default_context(); ctx.profile(True)
    B.sketch_product(a, x, transpose=True)
    B.sketch_product(a, r)
print(B.default_context().profile_report())
