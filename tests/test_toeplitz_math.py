"""The algebra behind the Toeplitz form of the correction solves
(paper_2010_05872_b200/csrc/fused3d.cu "Toeplitz solves",
api.cu:toeplitz_end_tables), restated in numpy: solving with the CONSTANT
Thomas factors w = 2 - sqrt(3), 1/d = 1/(4/3 - w/3) and adding the two
Sherman-Morrison end corrections reproduces batched_solve
(reference transform.hpp:116-130 with ThomasAux::build, :29-43) to rounding
for every line length the kernels use it on (m >= 40)."""
import numpy as np

LD = np.longdouble
OFF, DIAG_B, DIAG_I = 1.0 / 3.0, 2.0 / 3.0, 4.0 / 3.0
KTW = 2.0 - 1.7320508075688772
KTID = 1.0 / (DIAG_I - KTW * OFF)
ENDS = 32


def thomas_reference(f):
    m = len(f)
    d = DIAG_B
    w = np.zeros(m)
    inv = np.zeros(m)
    inv[0] = 1.0 / d
    for i in range(1, m):
        wi = OFF / d
        w[i] = wi
        d = (DIAG_B if i + 1 == m else DIAG_I) - wi * OFF
        inv[i] = 1.0 / d
    x = f.copy()
    for i in range(1, m):
        x[i] -= w[i] * x[i - 1]
    x[m - 1] *= inv[m - 1]
    for i in range(m - 2, -1, -1):
        x[i] = (x[i] - OFF * x[i + 1]) * inv[i]
    return x


def end_tables(m):
    w, idl, o = LD(KTW), LD(KTID), LD(OFF)
    d = 1 / idl
    a, b = d - LD(DIAG_B), w * o + d - LD(DIAG_B)
    y = np.zeros(m, dtype=LD)
    y[0] = 1
    for i in range(1, m):
        y[i] = -w * y[i - 1]
    g = np.zeros(m, dtype=LD)
    g[m - 1] = y[m - 1] * idl
    for i in range(m - 2, -1, -1):
        g[i] = (y[i] - o * g[i + 1]) * idl
    h = np.zeros(m, dtype=LD)
    h[m - 1] = idl
    for i in range(m - 2, -1, -1):
        h[i] = -o * idl * h[i + 1]
    ca, cb = a / (1 - a * g[0]), b / (1 - b * h[m - 1])
    gt = np.array([float(ca * g[k]) for k in range(ENDS)])
    ht = np.array([float(cb * h[m - 1 - k]) for k in range(ENDS)])
    return gt, ht


def toeplitz_solve(f):
    m = len(f)
    gt, ht = end_tables(m)
    z = f.copy()
    for i in range(1, m):
        z[i] = z[i] - KTW * z[i - 1]
    z[m - 1] *= KTID
    for i in range(m - 2, -1, -1):
        z[i] = (z[i] - OFF * z[i + 1]) * KTID
    x = z.copy()
    for k in range(ENDS):
        x[k] += z[0] * gt[k]
    for k in range(ENDS):
        x[m - 1 - k] += z[m - 1] * ht[k]
    return x


def test_constants_are_the_limit_of_the_thomas_factors():
    d = DIAG_B
    for _ in range(60):
        w = OFF / d
        d = DIAG_I - w * OFF
    assert abs(w - KTW) < 1e-16 and abs(1.0 / d - KTID) < 1e-16
    assert abs(KTW * KTW - 4.0 * KTW + 1.0) < 1e-15  # w^2 - 4 w + 1 = 0


def test_end_tables_decay_and_shape():
    gt, ht = end_tables(257)
    assert abs(gt[0] - 1.0) < 1e-15 and abs(ht[0] - 2.0 / np.sqrt(3.0)) < 1e-15
    for k in range(1, ENDS):
        assert abs(gt[k] / gt[k - 1] + KTW) < 1e-14
        assert abs(ht[k] / ht[k - 1] + KTW) < 1e-14
    assert abs(gt[-1]) < 3e-18 and abs(ht[-1]) < 3e-18  # 32 entries reach below fp64 rounding


def test_toeplitz_solve_equals_thomas():
    rng = np.random.default_rng(3)
    for m in (40, 41, 57, 64, 65, 129, 257, 513, 1025):
        for _ in range(3):
            f = rng.standard_normal(m) * 10.0 ** rng.integers(-3, 4)
            want = thomas_reference(f)
            got = toeplitz_solve(f)
            assert np.max(np.abs(got - want)) <= 6e-16 * np.max(np.abs(want)), m
