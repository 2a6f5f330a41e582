"""c3-shaped 3×FP16 range-finder passes (A·X and AᵀX, N = 60), timed by the library's
per-kernel CUDA events.  BCUR_UMMA_DEBUG (2 skip drain, 4 skip MMAs) isolates the data path."""
import sys, os, time, json
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
from paper_1703_06065_b200 import bcur as B
m, n, N = int(os.environ.get("PM", "16384")), int(os.environ.get("PNN", "65536")), int(os.environ.get("PN", "60"))
a = B.DeviceMatrix.generate("lowrank", np.float32, m, n, seed=0, sigma=[1.0] * 8, noise=1e-4)
xs = np.asfortranarray(np.random.default_rng(1).standard_normal((n, N)))
q = np.asfortranarray(np.random.default_rng(2).standard_normal((m, N)))
for _ in range(2):
    B.structured_product(a, xs, h3=True)
    B.structured_product(a, q, transpose=True, h3=True)
ctx = B.default_context()
ctx.profile(True)
for _ in range(3):
    B.structured_product(a, xs, h3=True)
    B.structured_product(a, q, transpose=True, h3=True)
ctx.synchronize()
rep = ctx.profile_report()
out = {k: v for k, v in rep.items() if "h3" in k or "sumsq" in k}
print(os.environ.get("BCUR_UMMA_DEBUG", "0"), json.dumps(out))
