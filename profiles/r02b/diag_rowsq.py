"""Where does the c3-shaped Pythagoras residual lose 6.5e-6 (rel_err) against the oracle?
Feeds the ORACLE's Q_C to the GPU's product paths and compares ‖Q_CᵀA‖² per path."""
import sys, os
sys.path.insert(0, os.environ.get("GRAFT_REPO_ROOT", "/root/repo"))
import numpy as np
from oracle import bcur_oracle as O
from paper_1703_06065_b200 import bcur as B

for (m, n, noise, g) in [(2048, 8192, 3e-4, 8), (2048, 8192, 3e-4, 32), (4096, 16384, 3e-4, 8), (8192, 8192, 3e-4, 8)]:
    a = O.gen_lowrank(m, n, O.spectrum("pow:1.5", 50), noise, 0, dtype=np.float32)
    part = O.BlockPartition.equal_blocks(n, 128)
    ref = O.block_css(a, part, 50, g, O.Rng(0), p=10, q=2, mode=O.WITHOUT_REPLACEMENT)
    bn2 = O.block_norms2(a, part)
    qc, _ = O.column_basis(a, part, ref.plan.blocks(), np.float32, bn2)
    a64 = a.astype(np.float64)
    x = a64.T @ qc
    exact = float(np.sum(x * x))
    f16 = B.structured_product(a, np.asfortranarray(qc), rowsq_f16=True)
    h3 = B.structured_product(a, np.asfortranarray(qc), transpose=True, h3=True)
    tf = B.sketch_product(a, np.asfortranarray(qc), transpose=True, row_sumsq=True)
    got = B.block_css(a, B.BlockPartition.equal_blocks(n, 128), 50, g, B.Rng(0), p=10, q=2,
                      mode=B.SamplingMode.without_replacement, return_c=False)
    a2 = float(np.sum(bn2))
    print(f"m={m} n={n} g={g}: rel_err oracle {ref.rel_err:.10f} gpu {got.rel_err:.10f} "
          f"(d={got.rel_err / ref.rel_err - 1:+.2e}) path {got.residual_path}")
    for name, v in (("rowsq_f16", float(np.sum(f16))), ("h3 store", float(np.sum(h3 * h3))), ("x1 tf32", float(np.sum(tf)))):
        print(f"   {name:10s} ‖QᵀA‖² rel dev {v / exact - 1:+.3e}   → rel_err dev {np.sqrt((a2 - v) / (a2 - exact)) - 1:+.3e}")
    print(f"   oracle Q orth dev {np.max(np.abs(qc.T @ qc - np.eye(qc.shape[1]))):.2e}", flush=True)
