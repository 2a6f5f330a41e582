"""The reference's binary matrix format (io.cpp:105-137, io.hpp:13-14): "BCUR", u64 rows,
u64 cols, f64 row-major.  CPU: the oracle's restatement against independently built bytes
and the committed fixture, and the library's header parser (no device needed).  GPU: the
streamed device loader (full and column shards, fp64 exact / fp32 rounded, chunk
boundaries) and its ParseError cases, checked against the oracle loader."""
import os
import struct

import numpy as np
import pytest

from oracle import bcur_oracle as O

GOLDEN = os.path.join(os.path.dirname(__file__), "golden", "small.bcur")


def raw_bytes(a):
    return b"BCUR" + struct.pack("<QQ", *a.shape) + np.ascontiguousarray(a, dtype="<f8").tobytes()


def test_oracle_format_bytes(tmp_path):
    a = np.arange(12, dtype=np.float64).reshape(3, 4) * 0.5 - 1.0
    p = tmp_path / "a.bcur"
    O.save_matrix_binary(p, a)
    assert p.read_bytes() == raw_bytes(a)
    np.testing.assert_array_equal(O.load_matrix_binary(p), a)


def test_golden_fixture():
    a = O.load_matrix_binary(GOLDEN)
    assert a.shape == (5, 7)
    assert open(GOLDEN, "rb").read() == raw_bytes(a)
    # the fixture holds i - 2.5·j + 1/(1+i+j): row-major order is visible in the values
    i, j = np.meshgrid(np.arange(5), np.arange(7), indexing="ij")
    np.testing.assert_array_equal(a, i - 2.5 * j + 1.0 / (1 + i + j))


@pytest.mark.parametrize("case", ["magic", "header", "dims", "data", "nan", "missing"])
def test_oracle_parse_errors(tmp_path, case):
    p = tmp_path / "bad.bcur"
    good = raw_bytes(np.ones((4, 3)))
    if case == "magic":
        p.write_bytes(b"BCUX" + good[4:])
    elif case == "header":
        p.write_bytes(good[:10])
    elif case == "dims":
        p.write_bytes(b"BCUR" + struct.pack("<QQ", 0, 3))
    elif case == "data":
        p.write_bytes(good[:-8])
    elif case == "nan":
        p.write_bytes(raw_bytes(np.array([[1.0, np.nan], [2.0, 3.0]])))
    else:
        p = tmp_path / "absent.bcur"
    with pytest.raises(O.ParseError):
        O.load_matrix_binary(p)


def test_library_header(tmp_path):
    from paper_1703_06065_b200 import bcur as B
    assert B.bcur_header(GOLDEN) == (5, 7)
    p = tmp_path / "bad.bcur"
    p.write_bytes(b"BCUR" + struct.pack("<QQ", 1 << 31, 2))
    with pytest.raises(B.ParseError):
        B.bcur_header(p)
    p.write_bytes(b"NOPE" + struct.pack("<QQ", 2, 2))
    with pytest.raises(B.ParseError):
        B.bcur_header(p)


@pytest.mark.gpu
@pytest.mark.parametrize("m,n,col0,ncols", [(37, 23, 0, -1), (3000, 2900, 0, -1), (3000, 2900, 700, 1000),
                                            (1, 5, 4, 1)])
def test_device_loader(tmp_path, m, n, col0, ncols):
    from paper_1703_06065_b200 import bcur as B
    a = np.random.default_rng(m + n).standard_normal((m, n)) * 10.0 ** np.random.default_rng(1).integers(-5, 5, n)
    p = tmp_path / "a.bcur"
    O.save_matrix_binary(p, a)
    ref = O.load_matrix_binary(p)
    hi = n if ncols < 0 else col0 + ncols
    d64 = B.DeviceMatrix.load_bcur(p, np.float64, col0, ncols)
    np.testing.assert_array_equal(d64.to_host(), ref[:, col0:hi])
    d32 = B.DeviceMatrix.load_bcur(p, np.float32, col0, ncols)
    np.testing.assert_array_equal(d32.to_host(), ref[:, col0:hi].astype(np.float32))
    q = tmp_path / "b.bcur"
    d64.save_bcur(q)
    assert q.read_bytes() == raw_bytes(ref[:, col0:hi])


@pytest.mark.gpu
@pytest.mark.parametrize("case", ["magic", "data", "nan", "range", "missing"])
def test_device_loader_errors(tmp_path, case):
    from paper_1703_06065_b200 import bcur as B
    p = tmp_path / "bad.bcur"
    good = raw_bytes(np.ones((40, 30)))
    exc = B.ParseError
    if case == "magic":
        p.write_bytes(b"XCUR" + good[4:])
    elif case == "data":
        p.write_bytes(good[:-100])
    elif case == "nan":
        a = np.ones((40, 30))
        a[39, 29] = np.inf
        p.write_bytes(raw_bytes(a))
    elif case == "range":
        p.write_bytes(good)
        exc = IndexError  # BCUR_E_OUT_OF_RANGE (std::out_of_range in the reference)
    else:
        p = tmp_path / "absent.bcur"
    with pytest.raises(exc):
        B.DeviceMatrix.load_bcur(p, np.float64, 25 if case == "range" else 0, 10 if case == "range" else -1)


@pytest.mark.gpu
def test_upload_async_orders_the_next_use():
    """bcur_dmat_upload_async: the copy runs on the upload stream; the next call that uses the
    matrix (here the norms pass, then a download) sees the new data; a second upload into the
    same matrix waits for the uses already enqueued."""
    import torch

    from paper_1703_06065_b200 import bcur as B

    gen = np.random.default_rng(7)
    m, n = 4096, 1536
    a1 = np.asfortranarray(gen.standard_normal((m, n)).astype(np.float32))
    a2 = np.asfortranarray(gen.standard_normal((m, n)).astype(np.float32) * 3)
    h1 = torch.from_numpy(a1.T.copy()).pin_memory()  # (n, m) row-major = column-major m × n
    h2 = torch.from_numpy(a2.T.copy()).pin_memory()
    d = B.DeviceMatrix.empty(np.float32, m, n)
    d.upload_async(h1.data_ptr(), m)
    assert abs(B.frobenius_norm(d) - np.linalg.norm(a1.astype(np.float64))) <= 1e-6 * np.linalg.norm(a1)
    d.upload_async(h2.data_ptr(), m)
    d.upload_async(h1.data_ptr(), m)
    d.upload_async(h2.data_ptr(), m)
    np.testing.assert_array_equal(d.to_host(), a2)
