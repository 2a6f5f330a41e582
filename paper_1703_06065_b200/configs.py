"""The five workloads of BASELINE.json "configs" (unspecified knobs filled per
SURVEY Appendix A, D5/D11; recorded in DESIGN.md §Workloads)."""
import numpy as np

CONFIGS = {
    # CPU-oracle smoke: fp64 500×2000, rank 10, σ_i = 10·0.8^i, ν = 1e-3, 100 blocks of 20
    "c1": dict(kind="lowrank", dtype="f64", m=500, n=2000, rank=10, spectrum="geom:10:0.8", noise=1e-3, s=20,
               k=10, p=5, q=0, mode="without_replacement", select="leverage", g=10, seed=0),
    # biometric-shaped: fp64 64×20000, 200 blocks of 100, greedy 8
    "c2": dict(kind="biometric", dtype="f64", m=64, n=20000, s=100, k=5, p=5, q=0, mode="without_replacement",
               select="greedy", g=8, seed=0),
    # fp32 16384×65536, rank 50 power law i^-1.5, ν = 1e-4, 512 blocks of 128, k=50 p=10 q=2, c=32
    "c3": dict(kind="lowrank", dtype="f32", m=16384, n=65536, rank=50, spectrum="pow:1.5", noise=1e-4, s=128,
               k=50, p=10, q=2, mode="without_replacement", select="leverage", g=32, seed=0),
    # fp32 32768², rank 100, 0.97^i, ν = 1e-3, 256×256 blocks of 128, k=100, 24 + 24 blocks, U = C⁺AR⁺
    "c4": dict(kind="lowrank", dtype="f32", m=32768, n=32768, rank=100, spectrum="geom:1:0.97", noise=1e-3, s=128,
               k=100, p=10, q=0, mode="without_replacement", select="cur", g=24, g_rows=24, seed=0),
    # fp32 65536×262144 (68.7 GB), rank 200, 1/i, ν = 1e-4, 2048 blocks of 128, k=200 p=20, c=64 + greedy 64
    "c5": dict(kind="lowrank", dtype="f32", m=65536, n=262144, rank=200, spectrum="pow:1", noise=1e-4, s=128,
               k=200, p=20, q=0, mode="without_replacement", select="leverage+greedy", g=64, seed=0),
}


def spectrum(spec: str, r: int) -> np.ndarray:
    kind, *args = spec.split(":")
    i = np.arange(r, dtype=np.float64)
    if kind == "geom":
        return float(args[0]) * float(args[1]) ** i
    if kind == "pow":
        return (i + 1.0) ** (-float(args[0]))
    raise ValueError(spec)
