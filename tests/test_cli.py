"""tools/bcur_b200 — the reference CLI's hot-path commands (tools/bcur_main.cpp decompose /
scores, plus css) over the library: exit codes and JSON errors on CPU; on a B200 the report
(serialize.cpp:110-122 schema) and the scores CSV (io.cpp:196-210) against the oracle."""
import csv
import io
import json
import os
import subprocess

import numpy as np
import pytest

from oracle import bcur_oracle as O

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
CLI = os.path.join(ROOT, "tools", "bcur_b200")


@pytest.fixture(scope="module")
def cli():
    from paper_1703_06065_b200 import build as b
    b.build()
    return CLI


def run(cli, *args):
    return subprocess.run([cli, *map(str, args)], capture_output=True, text=True, timeout=300)


def test_help_and_errors(cli, tmp_path):
    assert run(cli, "--help").returncode == 0
    r = run(cli, "decompose", "--input", tmp_path / "absent.bcur", "--block-size", 4)
    assert r.returncode == 2 and json.loads(r.stderr)["error"]["type"] == "ParseError"
    bad = tmp_path / "bad.bcur"
    bad.write_bytes(b"NOPE" + bytes(16))
    r = run(cli, "scores", "--input", bad, "--block-size", 4, "--k", 2)
    assert r.returncode == 2 and "magic" in json.loads(r.stderr)["error"]["message"]
    r = run(cli, "frobnicate")
    assert r.returncode == 2 and json.loads(r.stderr)["error"]["type"] == "InvalidArgument"


def matrix(tmp_path, m=120, n=600, seed=4):
    g = np.random.default_rng(seed)
    a = g.standard_normal((m, 8)) @ g.standard_normal((8, n)) + 1e-3 * g.standard_normal((m, n))
    p = tmp_path / "a.bcur"
    O.save_matrix_binary(p, a)
    return p, a


@pytest.mark.gpu
def test_decompose_report(cli, tmp_path):
    p, a = matrix(tmp_path)
    r = run(cli, "decompose", "--input", p, "--block-size", 30, "--k", 5, "--r", 24, "--g", 4, "--t", 3, "--seed", 7,
            "--out-dir", tmp_path / "out")
    assert r.returncode == 0, r.stderr
    rep = json.loads(r.stdout)
    assert list(rep) == ["schema_version", "shapes", "row_plan", "block_plan", "metrics", "trial_errors", "config"]
    part = O.BlockPartition.equal_blocks(600, 30)
    best, errs = O.block_cur_alg1_boosted(a, part, 5, 24, 4, 3, O.Rng(7))
    assert [d["row"] for d in rep["row_plan"]["draws"]] == [d.row for d in best.rows]
    assert [d["block"] for d in rep["block_plan"]["draws"]] == best.plan.blocks()
    np.testing.assert_allclose(rep["trial_errors"], errs, rtol=1e-6, atol=1e-9 * best.a_norm)
    assert rep["metrics"][0]["variant"] == "U" and rep["metrics"][1]["variant"] == "U_k"
    assert rep["metrics"][0]["abs_err"] == pytest.approx(best.abs_err_u, rel=1e-6, abs=1e-9 * best.a_norm)
    assert rep["shapes"]["U"] == [best.u.shape[0], 24]
    u = O.load_matrix_binary(tmp_path / "out" / "U.bcur")
    assert np.max(np.abs(u - best.u)) <= 1e-6 * np.max(np.abs(best.u))
    assert json.loads((tmp_path / "out" / "report.json").read_text()) == rep


@pytest.mark.gpu
def test_scores_csv(cli, tmp_path):
    p, a = matrix(tmp_path, seed=5)
    r = run(cli, "scores", "--input", p, "--block-size", 50, "--k", 6, "--seed", 3)
    assert r.returncode == 0, r.stderr
    lines = r.stdout.splitlines()
    assert lines[0].startswith("# config=") and json.loads(lines[0][9:])["command"] == "scores"
    head = dict(line[2:].split("=", 1) for line in lines[1:5])
    rows = list(csv.DictReader(io.StringIO("\n".join(lines[5:]))))
    part = O.BlockPartition.equal_blocks(600, 50)
    sub = O.range_finder(a, 6, 10, 2, O.omega_key_from_seed(3))
    ref = O.block_leverage(sub.v_k, part)
    np.testing.assert_allclose([float(x["score"]) for x in rows], ref.scores, rtol=1e-9)
    assert float(head["normalizer"]) == ref.normalizer
    assert float(head["block_stable_rank"]) == pytest.approx(O.block_stable_rank(sub.v_k, part), rel=1e-8)
    assert float(head["incoherence"]) == pytest.approx(O.incoherence(sub.u_k), rel=1e-8)
