"""The verify / bench command line in the reference's schema (reference cli.py)."""

import csv
import io
import contextlib

import numpy as np
import pytest

from paper_2601_14466_b200 import cli


@pytest.mark.parametrize("argv", [
    ["verify", "--routine", "syevd", "--n", "8"],
    ["verify", "--routine", "potrs", "--n", "8", "--mode", "mpmd"],
    ["verify", "--routine", "potrs", "--n", "8", "--trace", "t.csv"],
    ["verify", "--routine", "potrs", "--n", "8", "--matrix", "file:x.bcmg"],
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
