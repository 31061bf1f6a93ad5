"""The eigensolver oracle (oracle/bcmg_oracle.py: syevd_dense) pinned to the
reference's own eigh_hermitian outputs (tests/golden/eigen_golden.npz, made by
oracle/gen_golden_eigen.py).  CPU only.

The reference sums y = A v device by device, so its bits depend on the device
count; agreement is to the reference's own invariance tolerance
(test_acceptance.py:249-268: 10 n eps after phase alignment) on separated
spectra and to its quality bounds (test_acceptance.py:223-241: 100 n eps
residual and orthonormality) everywhere."""

import os

import numpy as np
import pytest

from conftest import GOLDEN
from oracle import bcmg_oracle as O

G = np.load(os.path.join(GOLDEN, "eigen_golden.npz"))
CASES = sorted({k.split("__")[0] for k in G.files})


def _eps(dt):
    return float(np.finfo(np.float32 if dt in (np.float32, np.complex64) else np.float64).eps)


@pytest.mark.parametrize("name", CASES)
def test_oracle_matches_reference(name):
    a, w_ref, v_ref, cfg = (G[f"{name}__{k}"] for k in ("a", "w", "v", "cfg"))
    n = a.shape[0]
    w, v = O.syevd_dense(a, int(cfg[1]))
    eps = _eps(a.dtype)
    scale = max(1.0, float(np.max(np.abs(w_ref))))
    assert w.dtype == w_ref.dtype
    assert np.max(np.abs(w.astype(np.float64) - w_ref)) <= 10 * n * eps * scale
    assert np.all(np.diff(w) >= 0)
    wide = np.complex128 if np.iscomplexobj(a) else np.float64
    a64, v64 = a.astype(wide), v.astype(wide)
    bound = 100 * n * eps
    assert np.linalg.norm(a64 @ v64 - v64 * w.astype(np.float64)) / np.linalg.norm(a64) <= bound
    assert np.linalg.norm(v64.conj().T @ v64 - np.eye(n)) <= bound
    if name.startswith("sep") or name in ("diag3", "hand2"):
        # simple, separated spectrum: the normalised eigenvectors are unique
        assert np.max(np.abs(v.astype(wide) - v_ref.astype(wide))) <= 10 * n * eps * 10


def test_oracle_phase_convention():
    name = "rand12_f64"
    w, v = O.syevd_dense(G[f"{name}__a"], 4)
    for k in range(v.shape[1]):
        anchor = v[np.argmax(np.abs(v[:, k])), k]
        assert anchor > 0


def test_oracle_convergence_budget():
    d = np.array([1.0, 2.0, 3.0])
    e = np.array([1.0, 1.0])
    with pytest.raises(O.ConvergenceError):
        O.tridiag_eig(d, e, max_iter=0)
