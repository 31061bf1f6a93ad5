"""The verify / bench command line in the reference's schema (reference cli.py)."""

import csv
import io
import contextlib

import numpy as np
import pytest

from paper_2601_14466_b200 import cli


@pytest.mark.parametrize("argv", [
    ["verify", "--routine", "potrs", "--n", "8", "--trace", "t.csv"],
    ["verify", "--routine", "potrs", "--n", "8", "--matrix", "nonsense"],
    ["gen", "--kind", "diag", "--n", "0", "--out", "x.bcmg"],
    ["bench", "--routine", "potri", "--n", "8", "--devices", "0"],
    ["bench", "--routine", "potrs", "--n", "8", "--reps", "0"],
])
def test_configuration_errors_exit_2(argv):
    """Out-of-scope and invalid configurations are configuration errors (cli.py:462-482)."""
    err = io.StringIO()
    with contextlib.redirect_stderr(err):
        assert cli.main(argv) == 2
    assert "configuration error" in err.getvalue()


def test_reference_generator_and_columns():
    """random_spd is B B^H + n I from Philox(key=seed) (cli.py:81-103); CSV columns
    start with the reference's BENCH_COLUMNS (cli.py:65-68)."""
    from paper_2601_14466_b200.core import ElementType

    a = cli.make_matrix("random_spd", 12, ElementType.real64, 3)
    gen = np.random.Generator(np.random.Philox(key=3))
    b = gen.uniform(-1.0, 1.0, (12, 12))
    ref = b @ b.T + 12 * np.eye(12)
    assert np.array_equal(a, (ref + ref.T) / 2)
    d = cli.make_matrix("diag", 5, ElementType.complex64, 1)
    assert d.dtype == np.complex64 and np.array_equal(np.diag(d).real, np.arange(1, 6))
    assert cli.BENCH_COLUMNS == ["routine", "n", "tile", "devices", "dtype", "mode", "rep", "alloc_seconds",
                                 "solve_seconds", "residual"]


@pytest.mark.gpu
def test_verify_passes_on_gpu(capsys):
    assert cli.main(["verify", "--routine", "potrs", "--n", "256", "--tile", "32,64", "--devices", "1,2"]) == 0
    out = capsys.readouterr().out.splitlines()
    assert len(out) == 8 and all(line.startswith("PASS ") for line in out)
    assert cli.main(["verify", "--routine", "potri", "--n", "128", "--matrix", "random_spd", "--dtype", "c128",
                     "--tile", "32", "--devices", "3"]) == 0
    assert all(line.startswith("PASS inverse-residual") for line in capsys.readouterr().out.splitlines())
    assert cli.main(["verify", "--routine", "potrs", "--n", "512", "--matrix", "device_spd", "--dtype", "f32",
                     "--tile", "128", "--nrhs", "3"]) == 0


@pytest.mark.gpu
def test_bench_csv_on_gpu(tmp_path, capsys):
    out = tmp_path / "b.csv"
    assert cli.main(["bench", "--routine", "potrs", "--n", "512", "--tile", "128", "--devices", "1,2", "--reps", "2",
                     "--out", str(out)]) == 0
    rows = list(csv.reader(open(out)))
    assert rows[0][:10] == cli.BENCH_COLUMNS and len(rows) == 5
    for r in rows[1:]:
        assert float(r[9]) <= 100 * 512 * np.finfo(np.float64).eps and float(r[-1]) > 0


@pytest.mark.gpu
def test_gpu_residuals_match_host():
    """The 64-bit GPU residuals equal the reference's host formulas (cli.py:113-125)."""
    from oracle import bcmg_oracle as O

    rng = np.random.default_rng(0)
    a = O.make_matrix("random_spd", 64, np.complex128, 2)
    x = rng.standard_normal((64, 2)) + 1j * rng.standard_normal((64, 2))
    b = a @ x + 1e-9 * rng.standard_normal((64, 2))
    assert cli.solve_residual(a, x, b) == pytest.approx(O.solve_residual(a, x, b), rel=1e-6)
    inv = np.linalg.inv(a) + 1e-10
    assert cli.inverse_residual(a, inv) == pytest.approx(O.inverse_residual(a, inv), rel=1e-6)
    w, v = np.linalg.eigh(a)
    w = w + 1e-9
    host = np.linalg.norm(a @ v - v * w) / np.linalg.norm(a)
    assert cli.eigen_residual(a, w, v) == pytest.approx(host, rel=1e-6)
    assert cli.orthonormality_defect(v + 1e-9) == pytest.approx(
        np.linalg.norm((v + 1e-9).conj().T @ (v + 1e-9) - np.eye(64)), rel=1e-6)


def test_gen_writes_reference_format(tmp_path):
    """gen (cli.py:449-458) writes the reference's matrix file byte for byte:
    compare with a file the reference's own write_matrix produced."""
    from conftest import GOLDEN

    out = tmp_path / "a.bcmg"
    assert cli.main(["gen", "--kind", "random_spd", "--n", "5", "--dtype", "c64", "--seed", "2",
                     "--out", str(out)]) == 0
    assert out.read_bytes() == open(f"{GOLDEN}/ref_random_spd5_c64.bcmg", "rb").read()
    ones = tmp_path / "b.bcmg"
    assert cli.main(["gen", "--kind", "ones", "--n", "6", "--nrhs", "2", "--out", str(ones)]) == 0
    from paper_2601_14466_b200.core import read_matrix

    assert np.array_equal(read_matrix(ones), np.ones((6, 2)))


def test_bad_matrix_file_is_configuration_error(tmp_path):
    """MatrixFileError -> exit 2 (cli.py:471-473)."""
    bad = tmp_path / "bad.bcmg"
    bad.write_bytes(b"NOPE" + bytes(12))
    err = io.StringIO()
    with contextlib.redirect_stderr(err):
        assert cli.main(["verify", "--routine", "potrs", "--matrix", f"file:{bad}"]) == 2
    assert "configuration error" in err.getvalue()


@pytest.mark.gpu
def test_verify_syevd_on_gpu(capsys):
    """reference test_cli.py:44-60, 100-110: syevd verify lines."""
    assert cli.main(["verify", "--routine", "syevd", "--n", "32", "--tile", "4", "--devices", "2", "--dtype", "c128",
                     "--matrix", "random_spd"]) == 0
    lines = capsys.readouterr().out.splitlines()
    assert [ln.split()[1] for ln in lines] == ["eigen-residual", "orthonormal", "ascending"]
    assert all(ln.startswith("PASS") for ln in lines)
    assert cli.main(["verify", "--routine", "syevd", "--n", "64", "--tile", "16", "--devices", "2",
                     "--matrix", "diag"]) == 0
    lines = capsys.readouterr().out.splitlines()
    assert lines[-1].startswith("PASS diag-eigenvalues")


@pytest.mark.gpu
def test_verify_files_on_gpu(tmp_path, capsys):
    """reference test_cli.py:86-150: file: sources, --result-out, --rhs,
    --eigenvalues-out; not-positive-definite file -> exit 1 with the pivot."""
    from paper_2601_14466_b200.core import read_matrix, write_matrix

    bad = tmp_path / "bad.bcmg"
    write_matrix(bad, np.asfortranarray(np.diag([1.0, -1.0])))
    err = io.StringIO()
    with contextlib.redirect_stderr(err):
        assert cli.main(["verify", "--routine", "potrs", "--tile", "1", "--devices", "2",
                         "--matrix", f"file:{bad}"]) == 1
    assert "not positive definite: pivot=2" in err.getvalue()
    out_path = tmp_path / "x.bcmg"
    assert cli.main(["verify", "--routine", "potrs", "--n", "8", "--tile", "2", "--devices", "2", "--matrix", "diag",
                     "--result-out", str(out_path)]) == 0
    x = read_matrix(out_path)
    assert x.shape == (8, 1) and np.max(np.abs(x[:, 0] - 1.0 / np.arange(1.0, 9.0))) <= 1e-15
    rhs = tmp_path / "b.bcmg"
    write_matrix(rhs, np.asfortranarray(2.0 * np.ones((8, 1))))
    assert cli.main(["verify", "--routine", "potrs", "--n", "8", "--tile", "4", "--matrix", "diag",
                     "--rhs", str(rhs)]) == 0
    w_path = tmp_path / "w.bcmg"
    assert cli.main(["verify", "--routine", "syevd", "--n", "6", "--tile", "2", "--devices", "2", "--matrix", "diag",
                     "--eigenvalues-out", str(w_path)]) == 0
    assert np.allclose(read_matrix(w_path)[:, 0], np.arange(1.0, 7.0), atol=1e-12)
    a_path = tmp_path / "a.bcmg"
    assert cli.main(["gen", "--kind", "random_spd", "--n", "40", "--dtype", "f32", "--out", str(a_path)]) == 0
    assert cli.main(["verify", "--routine", "syevd", "--matrix", f"file:{a_path}", "--tile", "8"]) == 0
    capsys.readouterr()


def test_bogus_mode_env_is_configuration_error(monkeypatch):
    """BCMG_MODE outside {spmd, mpmd} exits 2 (reference test_cli.py:161-175)."""
    monkeypatch.setenv("BCMG_MODE", "bogus")
    err = io.StringIO()
    with contextlib.redirect_stderr(err):
        assert cli.main(["verify", "--routine", "potrs", "--n", "8", "--tile", "2", "--devices", "2",
                         "--matrix", "diag"]) == 2
    assert "configuration error" in err.getvalue()


@pytest.mark.gpu
@pytest.mark.parametrize("routine", ["potrs", "potri", "syevd"])
def test_mode_flag_and_env_same_output(capsys, monkeypatch, routine):
    """--mode mpmd (isolated workers: one session and one shard allocation per
    device, shards reached through the transport's handle exchange) prints the
    same PASS lines as $BCMG_MODE=mpmd and as spmd, and writes the same bits
    (reference test_cli.py:161-175)."""
    import os
    import tempfile

    from paper_2601_14466_b200.core import read_matrix

    outs, results = [], []
    for mode, env in (("mpmd", None), (None, "mpmd"), ("spmd", None)):
        if env:
            monkeypatch.setenv("BCMG_MODE", env)
        else:
            monkeypatch.delenv("BCMG_MODE", raising=False)
        path = os.path.join(tempfile.mkdtemp(), "r.bcmg")
        argv = ["verify", "--routine", routine, "--n", "96", "--tile", "8", "--devices", "4", "--dtype", "c128",
                "--matrix", "random_spd", "--result-out", path] + (["--mode", mode] if mode else [])
        assert cli.main(argv) == 0
        outs.append(capsys.readouterr().out)
        results.append(read_matrix(path))
    assert outs[0] == outs[1] and "PASS" in outs[0]
    assert np.array_equal(results[0], results[1])
    assert np.array_equal(results[0], results[2]), "mpmd and spmd must give the same bits"
