"""CPU oracle for the block-cyclic Cholesky path -- TEST INFRASTRUCTURE ONLY.

This module restates, in numpy/scipy, the algorithm of the reference
(`bcmg`, /root/reference/pkg/src/bcmg) for the hot path named by
BASELINE.json's north star: the contiguous -> 1D block-cyclic column
redistribution, the tiled right-looking potrf, the tiled potrs
substitution and the tiled potri inverse.  Every function cites the
reference file:line it follows.

Who may use it: only ``tests/``, ``__graft_entry__.smoke()`` and
``bench.py``'s ``cpu_baseline`` / ``--impl reference`` leg -- always as the
checker or the timed CPU baseline, never as part of the product path.  The
product (``paper_2601_14466_b200``) never imports this file.

Pinning: the restatement is checked against golden vectors produced by the
reference itself (``oracle/gen_golden.py`` imports /root/reference and writes
``tests/golden/``), see ``tests/test_oracle_golden.py``.
"""

from __future__ import annotations

import math

import numpy as np
from scipy.linalg import solve_triangular

# --------------------------------------------------------------------------
# element types (reference core.py:61-121)
# --------------------------------------------------------------------------

DTYPE_CODES = {  # core.py:69-72: real32=0, real64=1, complex64=2, complex128=3
    np.dtype("<f4"): 0,
    np.dtype("<f8"): 1,
    np.dtype("<c8"): 2,
    np.dtype("<c16"): 3,
}


def eps_of(dtype) -> float:
    """Machine epsilon of the matching real width (core.py:96-99)."""
    dt = np.dtype(dtype)
    real = np.float32 if dt in (np.dtype("<f4"), np.dtype("<c8")) else np.float64
    return float(np.finfo(real).eps)


# --------------------------------------------------------------------------
# layout (reference layout.py:82-256)
# --------------------------------------------------------------------------


def column_counts(n_cols: int, tile: int, ndev: int) -> list[int]:
    """Columns per device under the 1D block-cyclic deal (layout.py:82-95)."""
    counts = [0] * ndev
    n_tiles = -(-n_cols // tile)
    for t in range(n_tiles):
        counts[t % ndev] += min(tile, n_cols - t * tile)
    return counts


def column_offsets(n_cols: int, tile: int, ndev: int) -> list[int]:
    """Prefix sums of column_counts (layout.py:98-104)."""
    out, acc = [], 0
    for c in column_counts(n_cols, tile, ndev):
        out.append(acc)
        acc += c
    return out


def home_of(g: int, n_cols: int, tile: int, ndev: int) -> tuple[int, int]:
    """(device, local column) of global column g (layout.py:107-123)."""
    if not 0 <= g < n_cols:
        raise IndexError(g)
    t = g // tile
    return t % ndev, (t // ndev) * tile + g % tile


def dest_positions(n_cols: int, tile: int, ndev: int) -> np.ndarray:
    """dest_of[p] for the contiguous -> cyclic permutation (layout.py:126-145).

    Position p of the device-concatenated contiguous storage holds global
    column p; it moves to its cyclic home, counted in device order.
    """
    offs = np.asarray(column_offsets(n_cols, tile, ndev), dtype=np.int64)
    p = np.arange(n_cols, dtype=np.int64)
    t = p // tile
    return offs[t % ndev] + (t // ndev) * tile + p % tile


def cycles_of(dest: np.ndarray) -> list[tuple[int, ...]]:
    """Disjoint cycles of a bijection, fixed points dropped, each cycle
    starting at its smallest member, cycles in ascending head order
    (layout.py:148-172)."""
    dest = np.asarray(dest, dtype=np.int64)
    n = dest.shape[0]
    if not np.array_equal(np.sort(dest), np.arange(n)):
        raise ValueError("not a bijection")
    visited = np.zeros(n, dtype=bool)
    out = []
    for head in range(n):
        if visited[head]:
            continue
        visited[head] = True
        if dest[head] == head:
            continue
        cyc = [head]
        q = int(dest[head])
        while q != head:
            visited[q] = True
            cyc.append(q)
            q = int(dest[q])
        out.append(tuple(cyc))
    return out


def reverse_cycles(cycles) -> list[tuple[int, ...]]:
    """Inverse plan: keep each head, reverse the tail (layout.py:175-183)."""
    return [(c[0],) + tuple(c[:0:-1]) for c in cycles]


def rotate_in_place(cols: np.ndarray, cycles) -> list[tuple[int, int]]:
    """Apply cycles to the columns of ``cols`` (n_rows x n_cols) in place,
    following the reference's staging discipline (layout.py:234-250): save
    the head, shift backwards along the cycle, restore the saved head into
    cycle[1].  Returns the copy transcript as (src, dst) column pairs with
    -1 for the staging buffer, which tests audit for read-after-overwrite."""
    log = []
    for cyc in cycles:
        m = len(cyc)
        staged = cols[:, cyc[0]].copy()
        log.append((cyc[0], -1))
        for i in range(m - 1, 0, -1):
            cols[:, cyc[(i + 1) % m]] = cols[:, cyc[i]]
            log.append((cyc[i], cyc[(i + 1) % m]))
        cols[:, cyc[1]] = staged
        log.append((-1, cyc[1]))
    return log


def deal_columns(columns: np.ndarray, tile: int, ndev: int) -> np.ndarray:
    """Out-of-place redistribution by literally dealing tiles onto devices,
    no shared index arithmetic (oracle.py:172-215)."""
    n_cols = columns.shape[1]
    per_dev: list[list[int]] = [[] for _ in range(ndev)]
    for t in range(-(-n_cols // tile)):
        per_dev[t % ndev].extend(range(t * tile, min((t + 1) * tile, n_cols)))
    order = [g for lst in per_dev for g in lst]
    return np.asfortranarray(columns[:, order])


# --------------------------------------------------------------------------
# generators and residuals (reference cli.py:81-152)
# --------------------------------------------------------------------------


def make_matrix(kind: str, n: int, dtype, seed: int = 1) -> np.ndarray:
    """diag(1..n) or B B^H + n I with B ~ U[-1,1) from Philox(key=seed),
    exactly Hermitian (cli.py:86-103)."""
    dt = np.dtype(dtype)
    if kind == "diag":
        return np.asfortranarray(np.diag(np.arange(1, n + 1)).astype(dt))
    if kind == "random_spd":
        gen = np.random.Generator(np.random.Philox(key=seed))
        bm = gen.uniform(-1.0, 1.0, (n, n))
        if dt.kind == "c":
            bm = bm + 1j * gen.uniform(-1.0, 1.0, (n, n))
        a = bm @ bm.conj().T + n * np.eye(n)
        a = (a + a.conj().T) / 2
        return np.asfortranarray(a.astype(dt))
    raise ValueError(kind)


def _wide(x):
    x = np.asarray(x)
    return x.astype(np.complex128 if np.iscomplexobj(x) else np.float64)


def solve_residual(a, x, b) -> float:
    """||Ax-b||_F / (||A||_F ||x||_F + ||b||_F) at 64-bit (cli.py:113-118)."""
    a, x, b = _wide(a), _wide(x), _wide(b)
    if x.ndim == 1:
        x, b = x[:, None], b[:, None]
    num = np.linalg.norm(a @ x - b)
    den = np.linalg.norm(a) * np.linalg.norm(x) + np.linalg.norm(b)
    return float(num / den) if den else float(num)


def inverse_residual(a, inv) -> float:
    """||A X - I||_F / sqrt(n) (cli.py:121-125)."""
    a = _wide(a)
    n = a.shape[0]
    return float(np.linalg.norm(a @ _wide(inv) - np.eye(n)) / math.sqrt(n))


def residual_tol(dtype, n: int) -> float:
    return 100.0 * n * eps_of(dtype)  # cli.py:143-144


def elementwise_tol(dtype) -> float:
    return 1e-12 if eps_of(dtype) < 1e-10 else 1e-4  # cli.py:147-148


# --------------------------------------------------------------------------
# unblocked references (reference oracle.py:46-115)
# --------------------------------------------------------------------------


def cholesky_unblocked(a: np.ndarray) -> tuple[np.ndarray, int]:
    """Left-looking unblocked lower Cholesky reading the lower triangle;
    returns (L, info) with LAPACK 1-based info (oracle.py:46-63)."""
    n = a.shape[0]
    L = np.zeros_like(a, order="F")
    for j in range(n):
        row = L[j, :j]
        d = a[j, j].real - np.real(np.vdot(row, row))
        if not (d > 0.0) or not math.isfinite(d):
            return L, j + 1
        L[j, j] = math.sqrt(d)
        if j + 1 < n:
            L[j + 1:, j] = (a[j + 1:, j] - L[j + 1:, :j] @ row.conj()) / L[j, j]
    return L, 0


def solve_unblocked(a: np.ndarray, b: np.ndarray) -> np.ndarray:
    """x = A^-1 b by explicit forward / conjugate-backward substitution
    (oracle.py:66-94)."""
    L, info = cholesky_unblocked(a)
    if info:
        raise ArithmeticError(f"not positive definite at pivot {info}")
    y = (b if b.ndim == 2 else b[:, None]).astype(L.dtype, copy=True)
    n = L.shape[0]
    for i in range(n):
        if i:
            y[i] -= L[i, :i] @ y[:i]
        y[i] /= L[i, i]
    for i in range(n - 1, -1, -1):
        if i + 1 < n:
            y[i] -= L[i + 1:, i].conj() @ y[i + 1:]
        y[i] /= L[i, i].conj()
    return y if b.ndim == 2 else y[:, 0]


def inverse_unblocked(a: np.ndarray) -> np.ndarray:
    """A^-1 = W^H W with W = L^-1, symmetrised (oracle.py:97-115)."""
    L, info = cholesky_unblocked(a)
    if info:
        raise ArithmeticError(f"not positive definite at pivot {info}")
    n = L.shape[0]
    W = np.zeros_like(L, order="F")
    for j in range(n):
        W[j, j] = 1.0 / L[j, j]
        for i in range(j + 1, n):
            W[i, j] = -(L[i, j:i] @ W[j:i, j]) / L[i, i]
    inv = W.conj().T @ W
    return np.asfortranarray((inv + inv.conj().T) / 2)


# --------------------------------------------------------------------------
# tiled algorithms (reference solvers.py:322-594), on the dense matrix
# --------------------------------------------------------------------------
#
# The reference runs these tile loops over per-device shards; the
# arithmetic per tile depends only on the tile width, never on the device
# count (solvers.py:350-354), so restating them on the global column-major
# matrix gives the same numbers.


def _tile_ranges(n: int, tile: int):
    return [(k, k * tile, min((k + 1) * tile, n)) for k in range(-(-n // tile))]


def potrf_tiled(a: np.ndarray, tile: int) -> tuple[np.ndarray, int]:
    """Right-looking tiled Cholesky of the lower triangle (solvers.py:341-406).

    Per tile: unblocked factor of the diagonal block (solvers.py:322-338),
    panel solve A21 <- A21 L11^-H (solvers.py:381-386), trailing update of
    every later tile C_m -= P P[m rows]^H (solvers.py:395-405; restricted
    here to rows >= the tile start, which is all the lower triangle
    reads).  Returns (matrix with L in its lower triangle, info)."""
    w = np.array(a, order="F", copy=True)
    n = w.shape[0]
    tiles = _tile_ranges(n, tile)
    for k, s, e in tiles:
        blk = w[s:e, s:e]
        for j in range(e - s):  # solvers.py:326-338
            d = blk[j, j].real - np.vdot(blk[j, :j], blk[j, :j]).real
            if not (d > 0.0) or not math.isfinite(d):
                return w, s + j + 1
            ljj = math.sqrt(d)
            blk[j, j] = ljj
            if j + 1 < e - s:
                blk[j + 1:, j] = (blk[j + 1:, j] - blk[j + 1:, :j] @ blk[j, :j].conj()) / ljj
        if e == n:
            continue
        xh = solve_triangular(blk, w[e:, s:e].conj().T, lower=True, check_finite=False)
        w[e:, s:e] = xh.conj().T
        for m, ms, me in tiles[k + 1:]:
            p = w[ms:, s:e]
            w[ms:, ms:me] -= p @ w[ms:me, s:e].conj().T
    return w, 0


def potrs_tiled(fact: np.ndarray, b: np.ndarray, tile: int) -> np.ndarray:
    """Tiled forward L y = b then backward L^H x = y (solvers.py:430-474)."""
    n = fact.shape[0]
    x = np.array(b if b.ndim == 2 else b[:, None], dtype=fact.dtype, order="F")
    tiles = _tile_ranges(n, tile)
    for k, s, e in tiles:
        x[s:e] = solve_triangular(fact[s:e, s:e], x[s:e], lower=True, check_finite=False)
        if e < n:
            x[e:] -= fact[e:, s:e] @ x[s:e]
    for k, s, e in reversed(tiles):
        if e < n:
            x[s:e] -= fact[e:, s:e].conj().T @ x[e:]
        x[s:e] = solve_triangular(fact[s:e, s:e], x[s:e], lower=True, trans="C",
                                  check_finite=False)
    return x if b.ndim == 2 else x[:, 0]


def potri_tiled(fact: np.ndarray, tile: int) -> np.ndarray:
    """Full Hermitian inverse from the factor (solvers.py:487-594):
    W = L^-1 swept from the last tile backwards, A^-1 = W^H W swept
    forwards, lower triangle mirrored with an exactly real diagonal."""
    n = fact.shape[0]
    tiles = _tile_ranges(n, tile)
    W = np.tril(np.array(fact, order="F", copy=True))
    for k, s, e in reversed(tiles):  # solvers.py:525-545
        w11 = solve_triangular(W[s:e, s:e], np.eye(e - s, dtype=W.dtype), lower=True,
                               check_finite=False)
        if e < n:
            acc = np.tril(W[e:, e:]) @ W[e:, s:e]
            W[e:, s:e] = -(acc @ w11)
        W[s:e, s:e] = w11
    W = np.tril(W)
    inv = np.zeros_like(W, order="F")
    for j, js, je in tiles:  # solvers.py:547-562
        inv[js:, js:je] = W[js:, js:].conj().T @ W[js:, js:je]
    low = np.tril(inv, -1)
    out = low + low.conj().T  # solvers.py:564-593
    out[np.diag_indices(n)] = np.real(np.diagonal(inv))
    return np.asfortranarray(out)


def solve_pipeline(a: np.ndarray, b: np.ndarray, tile: int) -> np.ndarray:
    """solve_positive_definite's arithmetic (solvers.py:931-985)."""
    fact, info = potrf_tiled(a, tile)
    if info:
        raise ArithmeticError(f"not positive definite: pivot={info}")
    return potrs_tiled(fact, b, tile)


def invert_pipeline(a: np.ndarray, tile: int) -> np.ndarray:
    """invert_positive_definite's arithmetic (solvers.py:988-1016)."""
    fact, info = potrf_tiled(a, tile)
    if info:
        raise ArithmeticError(f"not positive definite: pivot={info}")
    return potri_tiled(fact, tile)


def potrs_flops(n: int, nrhs: int, complex_: bool = False) -> float:
    """Algorithmic flops N^3/3 + 2 N^2 N_RHS (x4 complex) -- SURVEY 8(d)."""
    f = n ** 3 / 3.0 + 2.0 * n * n * nrhs
    return 4.0 * f if complex_ else f


# --------------------------------------------------------------------------
# Hermitian eigendecomposition (reference solvers.py:597-910), dense form.
# The reference walks the tiles device by device; the arithmetic per column is
# the same for every device count up to the summation order of y = A v, so
# the oracle runs it on one dense matrix.
# --------------------------------------------------------------------------


class ConvergenceError(ArithmeticError):
    """core.py:57-58"""


def householder(x: np.ndarray):
    """(v, tau, beta) with v[0] = 1, H^H x = beta e1, beta real (solvers.py:600-623)."""
    v = np.zeros_like(x)
    v[0] = 1
    alpha = complex(x[0])
    tail = float(np.linalg.norm(x[1:])) if len(x) > 1 else 0.0
    if tail == 0.0 and alpha.imag == 0.0:
        return v, 0.0, alpha.real
    beta = -math.copysign(math.hypot(abs(alpha), tail), alpha.real or 1.0)
    if np.iscomplexobj(x):
        v[1:] = x[1:] / (alpha - beta)
        tau = (beta - alpha) / beta
    else:
        v[1:] = x[1:] / (alpha.real - beta)
        tau = (beta - alpha.real) / beta
    return v, tau, beta


def tridiagonalize(a: np.ndarray, tile: int):
    """Blocked Householder reduction to real tridiagonal form (solvers.py:666-780):
    lazy per-column panel update from the tile's U / W, y = sym(A_stale) v with
    the U / W correction, W = tau y - sigma v, one rank-2T trailing update per
    tile.  Returns (d, e, reflectors [(c, v, tau)])."""
    a = np.array(a, dtype=a.dtype, order="F", copy=True)
    n = a.shape[0]
    dt = a.dtype
    d = np.zeros(n, dtype=np.float64)
    e = np.zeros(max(n - 1, 0), dtype=np.float64)
    refl = []
    for _, start, stop in _tile_ranges(n, tile):
        tc = stop - start
        u = np.zeros((n, tc), dtype=dt)
        w = np.zeros((n, tc), dtype=dt)
        for jj in range(tc):
            c = start + jj
            if jj:
                a[c:, c] -= u[c:, :jj] @ w[c, :jj].conj() + w[c:, :jj] @ u[c, :jj].conj()
            d[c] = a[c, c].real
            if c == n - 1:
                continue
            v, tau, beta = householder(np.array(a[c + 1:, c]))
            e[c] = beta
            refl.append((c, v, tau))
            if tau == 0:
                continue
            blk = a[c + 1:, c + 1:]
            low = np.tril(blk)
            y = low @ v + np.tril(blk, -1).conj().T @ v
            if jj:
                y -= u[c + 1:, :jj] @ (w[c + 1:, :jj].conj().T @ v) + w[c + 1:, :jj] @ (u[c + 1:, :jj].conj().T @ v)
            sigma = 0.5 * (abs(tau) ** 2) * np.vdot(v, y)
            u[c + 1:, jj] = v
            w[c + 1:, jj] = tau * y - sigma * v
        if stop < n:
            a[:, stop:] -= u @ w[stop:, :].conj().T + w @ u[stop:, :].conj().T
    return d, e, refl


def tridiag_eig(d_in, e_in, max_iter: int = 30):
    """Implicit-shift QL with Wilkinson shift, rotations accumulated into z
    (solvers.py:783-843)."""
    n = len(d_in)
    d = np.asarray(d_in, dtype=np.float64).copy()
    e = np.zeros(n, dtype=np.float64)
    e[: n - 1] = e_in[: n - 1] if n > 1 else 0.0
    z = np.eye(n)
    eps = np.finfo(np.float64).eps
    for l in range(n):
        iters = 0
        while True:
            for m in range(l, n - 1):
                if abs(e[m]) <= eps * (abs(d[m]) + abs(d[m + 1])):
                    break
            else:
                m = n - 1
            if m == l:
                break
            iters += 1
            if iters > max_iter:
                raise ConvergenceError(f"tridiagonal eigensolver exceeded {max_iter} iterations at index {l}")
            g = (d[l + 1] - d[l]) / (2.0 * e[l])
            r = math.hypot(g, 1.0)
            g = d[m] - d[l] + e[l] / (g + math.copysign(r, g))
            s = c = 1.0
            p = 0.0
            for i in range(m - 1, l - 1, -1):
                f = s * e[i]
                b = c * e[i]
                r = math.hypot(f, g)
                e[i + 1] = r
                if r == 0.0:
                    d[i + 1] -= p
                    e[m] = 0.0
                    break
                s = f / r
                c = g / r
                g = d[i + 1] - p
                r = (d[i] - g) * s + 2.0 * c * b
                p = s * r
                d[i + 1] = g + p
                g = c * r - b
                zi = z[:, i].copy()
                zi1 = z[:, i + 1].copy()
                z[:, i + 1] = s * zi + c * zi1
                z[:, i] = c * zi - s * zi1
            else:
                d[l] -= p
                e[l] = g
                e[m] = 0.0
    return d, z


def phase_normalize(v: np.ndarray) -> np.ndarray:
    """First largest-magnitude component of each column real and positive
    (solvers.py:898-909)."""
    v = np.array(v, copy=True)
    idx = np.argmax(np.abs(v), axis=0)
    lead = v[idx, np.arange(v.shape[1])]
    scale = np.abs(lead)
    safe = np.where(scale == 0, 1, scale)
    phase = np.where(scale == 0, 1, lead / safe)
    v *= np.conj(phase)[None, :]
    return v


def syevd_dense(a: np.ndarray, tile: int):
    """Eigenvalues ascending (real type of a) and phase-normalised eigenvectors
    (solvers.py:862-910 on one dense matrix)."""
    n = a.shape[0]
    dt = a.dtype
    d, e, refl = tridiagonalize(a, tile)
    w, z = tridiag_eig(d, e)
    order = np.argsort(w, kind="stable")
    w = w[order]
    z = np.asfortranarray(z[:, order].astype(dt))
    for c, v, tau in reversed(refl):
        if tau == 0:
            continue
        blk = z[c + 1:, :]
        blk -= tau * np.outer(v, v.conj() @ blk)
    real = np.float32 if dt in (np.float32, np.complex64) else np.float64
    return w.astype(real), phase_normalize(z)


def phase_align(v: np.ndarray, ref: np.ndarray) -> np.ndarray:
    """Scale each column of v by the unit phase that best matches ref
    (eigenvectors are unique only up to phase)."""
    dots = np.sum(v.conj() * ref, axis=0)
    mag = np.abs(dots)
    ph = np.where(mag == 0, 1, dots / np.where(mag == 0, 1, mag))
    return v * ph[None, :]
