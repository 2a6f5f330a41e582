"""Pins the oracle's Rng (and the product's C-ABI Rng) bit-for-bit against the
reference's own rng.hpp (rng.hpp:13-63), compiled by oracle/Makefile into
oracle/_ref/rng_dump, and against the C++ standard's mt19937_64 known answer."""
import os
import shutil
import struct
import subprocess

import pytest

from oracle import bcur_oracle as O

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
DUMP = os.path.join(ROOT, "oracle", "_ref", "rng_dump")
SEEDS = [0, 1, 42, 9001, (1 << 63) + 5]


def _ensure_dump():
    if not os.path.exists(DUMP) and os.path.isdir("/root/reference") and shutil.which("g++"):
        subprocess.run(["make", "-C", os.path.join(ROOT, "oracle")], check=True, capture_output=True)
    if not os.path.exists(DUMP):
        pytest.skip("oracle/_ref/rng_dump not built (reference sources absent on this host)")


def _hexd(x):
    return struct.pack(">d", x).hex()


def _ref_lines(seed, count):
    out = subprocess.run([DUMP, str(seed), str(count)], check=True, capture_output=True, text=True).stdout
    return out.strip().splitlines()


def _rng_lines(make_rng, seed, count):
    lines = []
    r = make_rng(seed)
    lines += [f"u64 {r.next_u64():016x}" for _ in range(count)]
    r = make_rng(seed)
    lines += [f"unif {_hexd(r.uniform01())}" for _ in range(count)]
    r = make_rng(seed)
    bounds = [1, 2, 3, 7, 10, 100, 1000003, 0x8000000000000001]
    lines += [f"below {bounds[i % 8]} {r.below(bounds[i % 8])}" for i in range(count)]
    r = make_rng(seed)
    lines += [f"normal {_hexd(r.normal())}" for _ in range(count)]
    r = make_rng(seed)
    lines += [f"split {s} {r.split(s).seed()}" for s in (0, 1, 2, 0x6F6D656761)]
    return lines


def test_mt19937_64_standard_known_answer():
    # C++ [rand.predef]: the 10000th invocation of a default-constructed mt19937_64
    e = O.MT19937_64(5489)
    for _ in range(9999):
        e()
    assert e() == 9981545732273789042


@pytest.mark.parametrize("seed", SEEDS)
def test_oracle_rng_matches_reference_rng_hpp(seed):
    _ensure_dump()
    assert _rng_lines(O.Rng, seed, 400) == _ref_lines(seed, 400)


@pytest.mark.parametrize("seed", SEEDS)
def test_product_rng_matches_reference_rng_hpp(seed):
    _ensure_dump()
    from paper_1703_06065_b200 import bcur
    assert _rng_lines(bcur.Rng, seed, 400) == _ref_lines(seed, 400)


def test_product_rng_matches_oracle_rng():
    from paper_1703_06065_b200 import bcur
    for seed in SEEDS:
        assert _rng_lines(bcur.Rng, seed, 50) == _rng_lines(O.Rng, seed, 50)
    assert bcur.omega_key(7) == O.omega_key_from_seed(7)
