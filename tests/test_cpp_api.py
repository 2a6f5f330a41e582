"""The header-only C++ mirror (include/bcur_b200.hpp): builds against the C ABI on any
host; on a B200 it runs the reference-style known-answer tests and config 1, whose
output must match tests/golden/c1.json."""
import json
import os
import shutil
import struct
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
PKG = os.path.join(ROOT, "paper_1703_06065_b200")
SRC = os.path.join(ROOT, "tests", "cpp", "test_cpp_api.cpp")


def build(tmp_path):
    if not shutil.which("g++"):
        pytest.skip("g++ not available")
    exe = str(tmp_path / "test_cpp_api")
    cmd = ["g++", "-std=c++20", "-O1", "-Wall", "-Wextra", "-I", os.path.join(ROOT, "include"), SRC, "-o", exe,
           "-L", PKG, "-lbcur_b200", f"-Wl,-rpath,{PKG}"]
    r = subprocess.run(cmd, capture_output=True, text=True)
    assert r.returncode == 0, r.stderr
    return exe


def test_cpp_mirror_compiles_and_links(tmp_path):
    build(tmp_path)


@pytest.mark.gpu
def test_cpp_mirror_runs_reference_style_tests(tmp_path):
    exe = build(tmp_path)
    r = subprocess.run([exe], capture_output=True, text=True, timeout=300)
    assert r.returncode == 0, r.stderr + r.stdout
    out = json.loads(r.stdout.strip().splitlines()[-1])
    with open(os.path.join(ROOT, "tests", "golden", "c1.json")) as f:
        g = json.load(f)
    d = lambda h: struct.unpack(">d", bytes.fromhex(h))[0]  # noqa: E731
    assert out["failures"] == 0
    assert out["blocks"] == g["plan"]["blocks"]
    assert out["normalizer"] == g["normalizer"]
    for got, ref in zip(out["scores"], g["scores"]):
        assert abs(got - d(ref)) <= 1e-9 * abs(d(ref))
    assert abs(out["abs_err"] - d(g["abs_err"])) <= 1e-6 * d(g["abs_err"])
