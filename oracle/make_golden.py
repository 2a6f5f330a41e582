"""Writes the committed golden fixtures under tests/golden/ — TEST INFRASTRUCTURE ONLY.

  rng_ref.json   the reference's own Rng (rng.hpp:13-63), run here through
                 oracle/_ref/rng_dump (built by oracle/Makefile from the reference
                 header); pins both the oracle's and the product's Rng on hosts
                 where /root/reference is absent (the GPU box).
  c1.json        config 1 (fp64 500×2000, 100 blocks of 20, k=10, p=5, c=10 w/o
                 replacement, seed 0): Philox-generated A checksums, block scores,
                 draws, margins, ‖A − CC⁺A‖_F — produced by the oracle.
  c2.json        config 2 (fp64 64×20000 biometric surrogate, greedy 8 of 200 blocks).
  c3s.json       config-3 structure at 2048×8192 fp32 (k=50, p=10, q=2, 8 of 64 blocks).
  c4s.json       config-4 structure at 1536×2048 fp32 (30, 4 col + 3 row blocks, U = C⁺AR⁺).
  c3.json        the headline config 3 itself (fp32 16384×65536, 32 of 512 blocks): written on
                 the GPU box by tests/test_gpu_zfullsize.py (the device-generated A downloaded
                 and run through the oracle; copied from gpurun_out/golden_c3.json).
  small.bcur     a 5×7 matrix (i − 2.5·j + 1/(1+i+j)) in the reference's binary format
                 (io.cpp:105-137), written by the oracle's save_matrix_binary.

The reference's numerical core (Eigen) cannot be built here, so everything but
rng_ref.json is oracle output: it freezes the oracle (tests re-derive it) and gives
the GPU parity tests a host-independent target.

Usage:  python -m oracle.make_golden      (from the repo root; needs oracle/_ref/rng_dump)
"""
from __future__ import annotations

import json
import os
import struct
import subprocess
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from oracle import bcur_oracle as O  # noqa: E402

OUT = os.path.join(ROOT, "tests", "golden")
DUMP = os.path.join(ROOT, "oracle", "_ref", "rng_dump")
RNG_SEEDS = [0, 1, 42, 9001, (1 << 63) + 5]
RNG_COUNT = 64


def hexd(x: float) -> str:
    return struct.pack(">d", float(x)).hex()


def checksums(a: np.ndarray) -> dict:
    a64 = np.asarray(a, dtype=np.float64)
    return {"sum": hexd(float(np.sum(a64))), "sumsq": hexd(float(np.sum(a64 * a64))),
            "corner": [hexd(a64[0, 0]), hexd(a64[-1, -1])]}


def plan_json(plan) -> dict:
    return {"blocks": [d.block for d in plan.draws], "probability": [hexd(d.probability) for d in plan.draws],
            "scale": [hexd(d.scale) for d in plan.draws], "margins": [float(x) for x in plan.margins]}


def rng_ref() -> dict:
    if not os.path.exists(DUMP):
        subprocess.run(["make", "-C", os.path.join(ROOT, "oracle")], check=True)
    out = {}
    for seed in RNG_SEEDS:
        txt = subprocess.run([DUMP, str(seed), str(RNG_COUNT)], check=True, capture_output=True, text=True).stdout
        out[str(seed)] = txt.strip().splitlines()
    return {"source": "oracle/_ref/rng_dump (reference rng.hpp)", "count": RNG_COUNT, "streams": out}


def lowrank(m, n, r, spec, noise, seed, dt):
    return O.gen_lowrank(m, n, O.spectrum(spec, r), noise, seed, dtype=dt)


def css_case(a, s, k, p, q, g, mode, seed) -> dict:
    part = O.BlockPartition.equal_blocks(a.shape[1], s)
    res = O.block_css(a, part, k, g, O.Rng(seed), p=p, q=q, mode=mode)
    return {"dtype": str(a.dtype), "m": a.shape[0], "n": a.shape[1], "s": s, "k": k, "p": p, "q": q, "g": g,
            "mode": mode, "seed": seed, "a": checksums(a),
            "scores": [hexd(x) for x in res.scores.scores], "normalizer": res.scores.normalizer,
            "plan": plan_json(res.plan), "abs_err": hexd(res.abs_err), "a_norm": hexd(res.a_norm),
            "rank_c": res.rank_c, "residual_path": res.residual_path}


def small_bcur():
    i, j = np.meshgrid(np.arange(5), np.arange(7), indexing="ij")
    O.save_matrix_binary(os.path.join(OUT, "small.bcur"), i - 2.5 * j + 1.0 / (1 + i + j))


def main():
    os.makedirs(OUT, exist_ok=True)
    small_bcur()
    files = {"rng_ref.json": rng_ref()}
    c = O.CONFIGS["c1"]
    a = lowrank(c["m"], c["n"], c["rank"], c["spectrum"], c["noise"], c["seed"], np.float64)
    files["c1.json"] = dict(css_case(a, c["s"], c["k"], c["p"], c["q"], c["g"], c["mode"], c["seed"]),
                            config="c1", spectrum=c["spectrum"], rank=c["rank"], noise=c["noise"])
    c = O.CONFIGS["c2"]
    a = O.gen_biometric(c["m"], c["n"], c["seed"])
    part = O.BlockPartition.equal_blocks(c["n"], c["s"])
    gr = O.greedy_select(a, part, c["k"], c["g"], O.omega_key_from_seed(c["seed"]), p=c["p"], q=c["q"])
    files["c2.json"] = {"config": "c2", "m": c["m"], "n": c["n"], "s": c["s"], "k": c["k"], "p": c["p"],
                        "q": c["q"], "g": c["g"], "seed": c["seed"], "a": checksums(a),
                        "steps": [{"block": st.block, "score": hexd(st.score), "margin": float(st.margin),
                                   "saturated": bool(st.saturated), "rank_added": int(st.rank_added)}
                                  for st in gr.steps],
                        "abs_err": hexd(gr.abs_err), "a_norm": hexd(gr.a_norm)}
    a = lowrank(2048, 8192, 50, "pow:1.5", 1e-4, 0, np.float32)
    files["c3s.json"] = dict(css_case(a, 128, 50, 10, 2, 8, O.WITHOUT_REPLACEMENT, 0), config="c3-scaled",
                             spectrum="pow:1.5", rank=50, noise=1e-4, data_seed=0)
    a = lowrank(1536, 2048, 40, "geom:1:0.97", 1e-3, 2, np.float32)
    co, ro = O.BlockPartition.equal_blocks(2048, 128), O.BlockPartition.equal_blocks(1536, 128)
    cur = O.block_cur_rows_cols(a, co, ro, 30, 4, 3, O.Rng(11), p=10)
    files["c4s.json"] = {"config": "c4-scaled", "m": 1536, "n": 2048, "rank": 40, "spectrum": "geom:1:0.97",
                         "noise": 1e-3, "data_seed": 2, "s": 128, "k": 30, "p": 10, "g": 4, "g_rows": 3,
                         "seed": 11, "a": checksums(a),
                         "col_scores": [hexd(x) for x in cur.col_scores.scores],
                         "row_scores": [hexd(x) for x in cur.row_scores.scores],
                         "col_plan": plan_json(cur.col_plan), "row_plan": plan_json(cur.row_plan),
                         "u_shape": list(cur.u.shape), "u_fro": hexd(float(np.linalg.norm(cur.u))),
                         "abs_err": hexd(cur.abs_err), "a_norm": hexd(cur.a_norm)}
    for name, obj in files.items():
        with open(os.path.join(OUT, name), "w") as f:
            json.dump(obj, f, indent=1)
            f.write("\n")
        print("wrote", os.path.join("tests", "golden", name))


if __name__ == "__main__":
    main()
