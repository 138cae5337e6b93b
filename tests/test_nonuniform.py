"""Pins of the nonuniform-coordinate restatement.

The reference has no nonuniform path, so the oracle's generalisation
(oracle/mgrx_oracle.c: nu_build — tensor-product linear interpolation
weights, fine mass matrix h/6, (h_l+h_r)/3 restricted by the coarse hats,
coarse mass matrix (H_{i-1}+H_i)/3, H_i/6) is pinned here against
first-principles checks written independently of it, following the
reference's own test oracles (proj/tests/oracles.hpp:22-45 quadrature,
:77-103 dense solve) with real node positions:

  1. equispaced coordinates reproduce the uniform path (bitwise equal to
     the reference) to <= 1e-13 * range;
  2. the load vector equals exact Gauss quadrature of (piecewise-linear
     interpolant) x (coarse hat) with real spacings, to 1e-12;
  3. the correction solve equals a dense solve of the nonuniform coarse
     mass matrix, to 1e-10;
  4. multilinear functions of the coordinates have zero coefficients;
  5. decompose -> recompose round-trips to 1e-9 * range.
"""
import numpy as np
import pytest

from oracle.oracle import Oracle
from synthetic_fields import nonuniform_coords


@pytest.fixture(scope="module")
def o():
    return Oracle()


def _quadrature_load(line, x):
    """f_i = integral of u * phi_i over the line, u the piecewise-linear
    interpolant of `line` on nodes x, phi_i the hat of coarse node x[2i]
    (support [x[2i-2], x[2i+2]]).  Two-point Gauss per fine cell is exact
    (the integrand is quadratic on each cell).  Odd lengths only."""
    n = len(x)
    m = (n + 1) // 2
    X = x[0::2]
    g = 1.0 / np.sqrt(3.0)
    out = np.zeros(m)
    for i in range(m):
        def hat(t):
            if i > 0 and X[i - 1] <= t <= X[i]:
                return (t - X[i - 1]) / (X[i] - X[i - 1])
            if i + 1 < m and X[i] <= t <= X[i + 1]:
                return (X[i + 1] - t) / (X[i + 1] - X[i])
            return 1.0 if t == X[i] else 0.0
        lo = X[i - 1] if i > 0 else X[i]
        hi = X[i + 1] if i + 1 < m else X[i]
        s = 0.0
        for cell in range(n - 1):
            a, b = x[cell], x[cell + 1]
            if b <= lo or a >= hi:
                continue
            for t in (0.5 * (1 - g), 0.5 * (1 + g)):
                xx = a + t * (b - a)
                u = line[cell] + (line[cell + 1] - line[cell]) * t
                s += 0.5 * (b - a) * u * hat(xx)
        out[i] = s
    return out


def _dense_nu_solve(f, X):
    """Coarse mass matrix on nodes X: diag (H_{i-1}+H_i)/3, off H_i/6."""
    m = len(X)
    H = np.diff(X)
    A = np.zeros((m, m))
    for i in range(m):
        A[i, i] = ((H[i - 1] if i > 0 else 0.0) + (H[i] if i + 1 < m else 0.0)) / 3.0
        if i + 1 < m:
            A[i, i + 1] = A[i + 1, i] = H[i] / 6.0
    return np.linalg.solve(A, f)


def test_equispaced_matches_uniform(o):
    rng = np.random.default_rng(11)
    for dims in [(17,), (33, 9), (9, 17, 12), (8, 10, 6)]:
        x = rng.uniform(-1, 1, dims)
        coords = [np.linspace(0.0, 1.0, n) for n in dims]
        nu = o.decompose_nu(x, coords)
        un = o.decompose(x)
        rng_ = float(x.max() - x.min())
        assert np.max(np.abs(nu - un)) <= 1e-13 * rng_, dims


@pytest.mark.parametrize("n", [3, 5, 9, 17, 33])
def test_load_vector_matches_quadrature(o, n):
    rng = np.random.default_rng(n)
    x = nonuniform_coords(n, seed=n)
    line = rng.normal(size=n)
    got = o.load_vector_nu_1d(line, x)
    want = _quadrature_load(line, x)
    assert np.max(np.abs(got - want)) <= 1e-12 * max(1.0, np.max(np.abs(want)))


@pytest.mark.parametrize("m", [2, 3, 5, 17, 65])
def test_correction_solve_matches_dense(o, m):
    rng = np.random.default_rng(m)
    X = nonuniform_coords(m, seed=m + 100)
    f = rng.normal(size=m)
    got = o.solve_correction_nu_1d(f.copy(), X)
    want = _dense_nu_solve(f, X)
    assert np.max(np.abs(got - want)) <= 1e-10 * max(1.0, np.max(np.abs(want)))


def test_multilinear_fields_vanish(o):
    rng = np.random.default_rng(5)
    for dims in [(33,), (17, 9), (9, 9, 17)]:
        coords = [nonuniform_coords(n, seed=2, axis=a) for a, n in enumerate(dims)]
        grids = np.meshgrid(*coords, indexing="ij")
        f = np.full(dims, rng.normal())
        # every product of distinct coordinate axes: multilinear
        for mask in range(1, 1 << len(dims)):
            term = np.full(dims, rng.normal())
            for a in range(len(dims)):
                if mask >> a & 1:
                    term = term * grids[a]
            f = f + term
        buf = o.decompose_nu(f, coords)
        _, level_dims, _ = o.hierarchy(dims)
        coarse = int(np.prod(level_dims[0]))  # everything after the coarsest block is a coefficient
        assert np.max(np.abs(buf[coarse:])) <= 1e-12 * float(f.max() - f.min()), dims


def test_roundtrip(o):
    rng = np.random.default_rng(9)
    for dims in [(65,), (33, 17), (17, 9, 12)]:
        coords = [nonuniform_coords(n, seed=4, axis=a) for a, n in enumerate(dims)]
        x = rng.uniform(-3, 3, dims)
        buf = o.decompose_nu(x, coords)
        back = o.recompose_nu(buf, dims, coords)
        assert np.max(np.abs(back - x)) <= 1e-9 * float(x.max() - x.min()), dims
