"""SKMX matrix files (matrix.hpp:70-93, matrix.cpp:13-61): byte-identical to the
reference's writer, readable by the reference's reader, same error behaviour
(test_executor.cpp:186-199 restated)."""
import ctypes as C
import os

import numpy as np
import pytest


def test_roundtrip_and_header(sk, tmp_path, port):
    A = port.random_matrix(7, 9, 123, "float32")
    p = str(tmp_path / "a.skmx")
    sk.save_matrix(p, A)
    assert os.path.getsize(p) == 16 + 7 * 9 * 4
    raw = open(p, "rb").read()
    assert raw[:4] == b"SKMX" and int.from_bytes(raw[4:8], "little") == 1
    back = sk.load_matrix(p, sk.DType.Float32)
    assert back.shape == (7, 9) and np.array_equal(back, A)
    with pytest.raises(sk.MatrixFileError):
        sk.load_matrix(p, sk.DType.Float64)  # dtype tag mismatch
    open(p, "wb").write(b"XXXX" + raw[4:])
    with pytest.raises(sk.MatrixFileError):
        sk.load_matrix(p, sk.DType.Float32)  # bad magic
    open(p, "wb").write(raw[:20])
    with pytest.raises(sk.MatrixFileError):
        sk.load_matrix(p, sk.DType.Float32)  # truncated payload


def test_bytes_identical_to_reference(sk, ref, tmp_path):
    for name, dt, sd in (("f32", "float32", sk.DType.Float32), ("f64", "float64", sk.DType.Float64),
                         ("i64", "int64", sk.DType.Int64)):
        A = ref.random_matrix(13, 5, 77, dt)
        pr, po = str(tmp_path / f"r_{name}"), str(tmp_path / f"o_{name}")
        assert getattr(ref.lib, f"ref_save_matrix_{name}")(
            os.fsencode(pr), C.c_int64(13), C.c_int64(5), A.ctypes.data_as(C.c_void_p)) == 0
        sk.save_matrix(po, A)
        assert open(pr, "rb").read() == open(po, "rb").read()
        assert np.array_equal(sk.load_matrix(pr, sd), A)
    # the reference reads ours and rejects a dtype mismatch with runtime_error (7)
    A = ref.random_matrix(4, 6, 5, "float32")
    po = str(tmp_path / "x")
    sk.save_matrix(po, A)
    r, c = C.c_int64(), C.c_int64()
    buf = np.empty(24, np.float32)
    assert ref.lib.ref_load_matrix_f32(os.fsencode(po), C.byref(r), C.byref(c),
                                       buf.ctypes.data_as(C.c_void_p), C.c_int64(24)) == 0
    assert np.array_equal(buf.reshape(4, 6), A)
    sk.save_matrix(po, A.astype(np.float64))
    assert ref.lib.ref_load_matrix_f32(os.fsencode(po), C.byref(r), C.byref(c),
                                       buf.ctypes.data_as(C.c_void_p), C.c_int64(24)) == 7
