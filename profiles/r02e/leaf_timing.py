import sys, os
sys.path.insert(0, os.environ.get("GRAFT_REPO_ROOT", "/root/repo"))
import numpy as np
from paper_1703_06065_b200 import bcur as B
gen = np.random.default_rng(0)
for w in (128, 128, 96, 64):
    x = gen.standard_normal((w + 64, w))
    r, ri, info, mn = B.cholesky(np.asfortranarray(x.T @ x))
    print("w", w, "info", info, flush=True)
