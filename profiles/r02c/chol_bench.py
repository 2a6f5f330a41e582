"""Timing of the recursive Cholesky + inverse (bcur_cholesky) and of the DMMA fp64 GEMM."""
import sys, os, time
sys.path.insert(0, os.environ.get("GRAFT_REPO_ROOT", "/root/repo"))
import numpy as np
import torch
from paper_1703_06065_b200 import bcur as B

ctx = B.default_context()
gen = np.random.default_rng(0)
for w in [128, 512, 1024, 2048, 4096]:
    x = gen.standard_normal((w + 64, w))
    g = np.asfortranarray(x.T @ x)
    gd = B.DeviceMatrix.from_host(g)
    hs = []
    for _ in range(2):
        import ctypes as C
        h = C.c_void_p(); B._check(B.L.lib.bcur_dmat_create(ctx.handle, B.L.F64, w, w, C.byref(h))); hs.append(B.DeviceMatrix(h, ctx))
    info, mn = C.c_int(), C.c_double()
    for it in range(6):
        ctx.synchronize(); t0 = time.perf_counter()
        B._check(B.L.lib.bcur_cholesky(ctx.handle, gd.handle, hs[0].handle, hs[1].handle, C.byref(info), C.byref(mn)))
        ctx.synchronize(); t1 = time.perf_counter()
    print(f"cholesky+inverse w={w}: {1e3*(t1-t0):.3f} ms (host wall, synced) info={info.value}", flush=True)
# DMMA GEMM rate: sketch_product with an fp64 A (A·X)
for (m, n, N) in [(4096, 4096, 4096), (2048, 2048, 2048), (16384, 4096, 60), (8192, 8192, 128)]:
    a = B.DeviceMatrix.from_host(np.asfortranarray(gen.standard_normal((m, n))))
    xd = B.DeviceMatrix.from_host(np.asfortranarray(gen.standard_normal((n, N))))
    h = C.c_void_p(); B._check(B.L.lib.bcur_dmat_create(ctx.handle, B.L.F64, m, N, C.byref(h))); o = B.DeviceMatrix(h, ctx)
    for it in range(4):
        ctx.synchronize(); t0 = time.perf_counter()
        B._check(B.L.lib.bcur_sketch_product(ctx.handle, a.handle, xd.handle, 0, o.handle, None))
        ctx.synchronize(); t1 = time.perf_counter()
    print(f"dgemm {m}x{n}x{N}: {1e3*(t1-t0):.3f} ms  {2.0*m*n*N/(t1-t0)/1e12:.2f} TF/s", flush=True)
