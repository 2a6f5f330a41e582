"""Reference point only (not product code): library fp64 Cholesky + triangular inverse times."""
import torch, time
for n in (3072, 4096, 8192):
    a = torch.randn(n * 4, n, dtype=torch.float64, device="cuda")
    g = a.T @ a
    for _ in range(2):
        r = torch.linalg.cholesky(g, upper=True)
        ri = torch.linalg.solve_triangular(r, torch.eye(n, dtype=torch.float64, device="cuda"), upper=True)
    torch.cuda.synchronize()
    e0, e1, e2 = (torch.cuda.Event(enable_timing=True) for _ in range(3))
    e0.record()
    for _ in range(5):
        r = torch.linalg.cholesky(g, upper=True)
    e1.record()
    for _ in range(5):
        ri = torch.linalg.solve_triangular(r, torch.eye(n, dtype=torch.float64, device="cuda"), upper=True)
    e2.record()
    torch.cuda.synchronize()
    print(n, "potrf %.3f ms" % (e0.elapsed_time(e1) / 5), "trsm-inverse %.3f ms" % (e1.elapsed_time(e2) / 5))
