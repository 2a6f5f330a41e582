"""The C-ABI library loads on a GPU-less host and exports every entry point the
public headers declare (no compute calls here)."""
import ctypes
import glob
import os
import re
import subprocess

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
LIB = os.path.join(ROOT, "paper_1703_06065_b200", "libbcur_b200.so")


def declared_functions():
    names = set()
    for h in glob.glob(os.path.join(ROOT, "include", "*.h")):
        src = open(h).read()
        src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
        for m in re.finditer(r"^[A-Za-z_][\w \t\*]*?\b(bcur_\w+)\s*\(", src, flags=re.M):
            names.add(m.group(1))
    return sorted(names)


def test_header_declares_the_boundary():
    names = declared_functions()
    for required in ["bcur_ctx_create", "bcur_block_leverage", "bcur_column_leverage", "bcur_range_finder",
                     "bcur_draw_blocks", "bcur_materialize_columns", "bcur_error_report", "bcur_block_css",
                     "bcur_greedy_select", "bcur_block_cur", "bcur_frobenius_norm", "bcur_last_error"]:
        assert required in names, required


def test_library_exports_every_declared_symbol():
    assert os.path.exists(LIB), "build first: python -m paper_1703_06065_b200.build"
    lib = ctypes.CDLL(LIB)
    missing = [n for n in declared_functions() if not hasattr(lib, n)]
    assert not missing, missing
    out = subprocess.run(["nm", "-D", "--defined-only", LIB], capture_output=True, text=True, check=True).stdout
    exported = {line.split()[-1] for line in out.splitlines() if " T " in line}
    assert set(declared_functions()) <= exported


def test_version_and_error_string_without_gpu():
    lib = ctypes.CDLL(LIB)
    lib.bcur_version.restype = ctypes.c_char_p
    lib.bcur_last_error.restype = ctypes.c_char_p
    assert lib.bcur_version().decode().startswith("bcur_b200")
    assert isinstance(lib.bcur_last_error(), (bytes, type(None)))
