"""BCMG matrix file format (reference core.py:36-38, 255-303; tests
test_core.py:112-150), pinned to files written by the reference itself
(tests/golden/ref_*.bcmg, oracle/gen_golden_eigen.py).  CPU only."""

import numpy as np
import pytest

from conftest import ALL_DTYPES, GOLDEN
from paper_2601_14466_b200.core import MATRIX_FILE_MAGIC, MatrixFileError, read_matrix, write_matrix


@pytest.mark.parametrize("dtype", ALL_DTYPES)
def test_round_trip(tmp_path, dtype):
    rng = np.random.default_rng(3)
    a = rng.standard_normal((5, 3))
    if np.dtype(dtype).kind == "c":
        a = a + 1j * rng.standard_normal((5, 3))
    a = np.asfortranarray(a.astype(dtype))
    path = tmp_path / "m.bcmg"
    write_matrix(path, a)
    back = read_matrix(path)
    assert back.dtype == a.dtype and back.flags.f_contiguous and back.flags.writeable
    assert np.array_equal(back, a)
    assert path.stat().st_size == 16 + a.nbytes


def test_reference_written_files():
    a = read_matrix(f"{GOLDEN}/ref_random_spd5_c64.bcmg")
    assert a.dtype == np.complex64 and a.shape == (5, 5) and np.allclose(a, a.conj().T)
    v = read_matrix(f"{GOLDEN}/ref_vector3_f32.bcmg")
    assert v.shape == (3, 1) and np.array_equal(v[:, 0], np.array([1.5, -2.0, 3.25], np.float32))


def test_header_layout(tmp_path):
    path = tmp_path / "m.bcmg"
    write_matrix(path, np.eye(2, order="F"))
    raw = path.read_bytes()
    assert raw[:4] == MATRIX_FILE_MAGIC and raw[4] == 1 and raw[5:8] == b"\0\0\0"
    assert int.from_bytes(raw[8:12], "little") == 2 and int.from_bytes(raw[12:16], "little") == 2


@pytest.mark.parametrize("mutate", ["magic", "truncate_payload", "truncate_header", "code", "dims", "extra"])
def test_rejections(tmp_path, mutate):
    path = tmp_path / "m.bcmg"
    write_matrix(path, np.eye(4, order="F"))
    raw = bytearray(path.read_bytes())
    if mutate == "magic":
        raw[:4] = b"XXXX"
    elif mutate == "truncate_payload":
        raw = raw[:-8]
    elif mutate == "truncate_header":
        raw = raw[:10]
    elif mutate == "code":
        raw[4] = 9
    elif mutate == "dims":
        raw[8:12] = (0).to_bytes(4, "little")
    else:
        raw += b"\0" * 8
    path.write_bytes(bytes(raw))
    with pytest.raises(MatrixFileError):
        read_matrix(path)


def test_write_rejects_3d(tmp_path):
    with pytest.raises(ValueError):
        write_matrix(tmp_path / "m.bcmg", np.zeros((2, 2, 2)))
