import numpy as np, sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1703_06065_b200 import bcur as B
gen = np.random.default_rng(0)
m, n, N = 64, 128, 16
a = np.asfortranarray(gen.standard_normal((m, n)).astype(np.float32))
x = np.asfortranarray(gen.standard_normal((n, N)))
q = np.asfortranarray(gen.standard_normal((m, N)))
np.set_printoptions(precision=5, suppress=True, linewidth=150)
y = B.sketch_product(a, x); ref = a.astype(np.float64) @ x
print("AX got\n", y[:3, :6], "\nref\n", ref[:3, :6])
z = B.sketch_product(a, q, transpose=True); refz = a.astype(np.float64).T @ q
print("AtX got\n", z[:3, :6], "\nref\n", refz[:3, :6])
r = B.sketch_product(a, q, transpose=True, row_sumsq=True)
print("rowsq got", r[:4], "ref", np.sum(refz**2, axis=1)[:4])
# identity-like test: a = small ints, x = e_j
a2 = np.asfortranarray(np.arange(m*n).reshape(m, n, order="F").astype(np.float32) % 7)
x2 = np.zeros((n, N)); x2[0, 0] = 1; x2[1, 1] = 1; x2[5, 2] = 2
print("AX e:\n", B.sketch_product(a2, x2)[:4, :4], "\nref\n", (a2.astype(np.float64) @ x2)[:4, :4])
q2 = np.zeros((m, N)); q2[0, 0] = 1; q2[1, 1] = 1; q2[3, 2] = 2
print("AtX e:\n", B.sketch_product(a2, q2, transpose=True)[:4, :4], "\nref\n", (a2.astype(np.float64).T @ q2)[:4, :4])
print(B.default_context().launch_count)
