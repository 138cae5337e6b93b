"""BASELINE.json configurations at their full sizes on the GPU, checked
against the pinned CPU oracle (oracle/libmgrx_oracle.so, which is
bit-identical to the reference on the uniform path — tests/test_oracle.py)
on the same seeded synthetic inputs, plus the size-independent properties
the domain offers (round trip, quantization error bound).

  config 2   513^3 f32                    coefficients <= 1e-5 * range, labels,
                                          L_inf <= tau for tau in {1e-2,1e-3,1e-4} * range
  config 3   4097^2 f64, nonuniform       coefficients <= 1e-12 * range vs the
                                          nonuniform restatement; round trip
  config 4a  100 x 500 x 500 f32          coefficients, labels, L_inf <= tau
  config 4b  288 x 115 x 69 x 69 f32      coefficients (4-D: general path), labels
  config 5b  1025^3 f32 (> 2^30 elements) coefficients, labels, L_inf <= tau

Label bar: bit-exact except values whose CPU coefficient lies within 1 ulp
of a bin edge (counted, reported in the assertion message).  Quantizing the
oracle's own coefficients on the GPU must be bit-exact.  The budget rule
(SURVEY.md §8(d)): budget = tau / C with C = 4 (C = 2 is the survey's
recommendation; the reference itself exceeds tau with C = 2 on some fields,
see tests/cpp/test_dropin.cpp).
"""
import numpy as np
import pytest

pytestmark = [pytest.mark.gpu, pytest.mark.slow]
C_BUDGET = 4.0


@pytest.fixture(scope="module")
def torch():
    import torch as t

    return t


@pytest.fixture(scope="module")
def mg():
    import paper_2010_05872_b200 as m

    return m


@pytest.fixture(scope="module")
def o():
    from oracle.oracle import Oracle

    return Oracle()


def _edge_flips(mg, h, plan, want, got_labels, ref_labels):
    """Label differences; each must be within 1 ulp of a bin edge."""
    from oracle.parity import label_flips

    n, worst = label_flips(want, got_labels, ref_labels, h.delta_counts(), plan.bin_widths, ulps=1.0)
    return n


def _check_field(torch, mg, o, f, taus, tol):
    """decompose / recompose / quantize a field against the oracle."""
    fh = f.cpu().numpy()
    rg = float(fh.max() - fh.min())
    h = mg.GridHierarchy.create(f.shape)
    ws = mg.SolverWorkspace()
    mc = mg.decompose(f, h, 0, ws)
    got = mc.buffer.cpu().numpy()
    want = o.decompose(fh)
    err = float(np.max(np.abs(got.astype(np.float64) - want)))
    assert err <= tol * rg, ("decompose", err / rg)
    back = mg.recompose(mc, ws).cpu().numpy()
    wr = o.recompose(want.astype(fh.dtype), fh.shape)
    err = float(np.max(np.abs(back.astype(np.float64) - wr)))
    assert err <= tol * rg, ("recompose", err / rg)
    flips = []
    for t in taus:
        tau = t * rg
        plan = mg.make_plan(mg.QuantMode.levelwise, tau / C_BUDGET, h)
        # the oracle's coefficients quantized on the GPU: bit-exact
        wantT = want.astype(fh.dtype)
        s_o = mg.quantize(mg.MultilevelCoefficients(torch.from_numpy(wantT).cuda(), h, 0), plan, ws)
        lab, opos, oval = o.quantize(wantT, fh.shape, plan.bin_widths)
        assert np.array_equal(s_o.flat.cpu().numpy(), lab)
        assert np.array_equal(s_o.outlier_positions.cpu().numpy(), opos)
        # the GPU's own coefficients: flips only at bin edges
        s = mg.quantize(mc, plan, ws)
        flips.append(_edge_flips(mg, h, plan, wantT, s.flat.cpu().numpy(), lab))
        rec = mg.recompose(mg.dequantize(s, plan, h, ws), ws).cpu().numpy()
        linf = float(np.max(np.abs(rec.astype(np.float64) - fh)))
        assert linf <= tau, ("L_inf / tau", linf / tau)
    return flips


def test_config2_full_size(torch, mg, o):
    from synthetic_fields import config2_field

    f = config2_field(device="cuda")
    flips = _check_field(torch, mg, o, f, (1e-2, 1e-3, 1e-4), 1e-5)
    print("config2 bin-edge label flips at tau = 1e-2/1e-3/1e-4 * range:", flips)


def test_config5b_full_size(torch, mg, o):
    """Config 5b's single field, 1025^3 f32 (1.08e9 elements, above 2^30):
    the fused wide-row kernels against the oracle, coefficients and
    recompose <= 1e-5 * range, labels at tau = 1e-3 * range within 1 ulp of
    a bin edge, L_inf <= tau."""
    from synthetic_fields import config2_field

    f = config2_field((1025, 1025, 1025), seed=0, device="cuda")
    flips = _check_field(torch, mg, o, f, (1e-3,), 1e-5)
    print("config5b bin-edge label flips at tau = 1e-3 * range:", flips)


def test_config4a_full_size(torch, mg, o):
    from synthetic_fields import config4a_field

    f = config4a_field(device="cuda")
    print("config4a bin-edge label flips:", _check_field(torch, mg, o, f, (1e-3,), 1e-5))


def test_config4b_full_size(torch, mg, o):
    from synthetic_fields import config4b_field

    f = config4b_field(device="cuda")
    print("config4b bin-edge label flips:", _check_field(torch, mg, o, f, (1e-3,), 1e-5))


def test_config3_nonuniform_full_size(torch, mg, o):
    from synthetic_fields import config3_field

    f, coords = config3_field(device="cuda")
    fh = f.cpu().numpy()
    rg = float(fh.max() - fh.min())
    h = mg.GridHierarchy.create(f.shape)
    ws = mg.SolverWorkspace()
    mc = mg.decompose_nonuniform(f, h, coords, 0, ws)
    want = o.decompose_nu(fh, coords)
    assert float(np.max(np.abs(mc.buffer.cpu().numpy() - want))) <= 1e-12 * rg
    back = mg.recompose_nonuniform(mc, coords, ws).cpu().numpy()
    assert float(np.max(np.abs(back - fh))) <= 1e-9 * rg
    wr = o.recompose_nu(want, fh.shape, coords)
    assert float(np.max(np.abs(mg.recompose_nonuniform(mg.MultilevelCoefficients(
        torch.from_numpy(want).cuda(), h, 0), coords, ws).cpu().numpy() - wr))) <= 1e-12 * rg


@pytest.mark.parametrize("dtype", ["f64", "f32"])
def test_nonuniform_shapes(torch, mg, o, dtype):
    """Nonuniform path on 1-D..4-D shapes (odd/even extents, partial stop
    levels) against the restatement; equispaced coordinates reproduce the
    uniform GPU path to rounding."""
    from synthetic_fields import nonuniform_coords

    npdt = np.float64 if dtype == "f64" else np.float32
    tol = 1e-12 if dtype == "f64" else 1e-5
    rng = np.random.default_rng(3)
    ws = mg.SolverWorkspace()
    # (300, 258), (257, 130), (130, 301): the fused 2-D nonuniform passes
    # (>= 2^13 nodes) with even / odd extents on either axis
    for shape in [(65,), (64,), (33, 20), (17, 9, 12), (40, 36, 66), (9, 8, 7, 6), (300, 258), (257, 130), (130, 301)]:
        coords = [nonuniform_coords(n, seed=1, axis=a) for a, n in enumerate(shape)]
        x = rng.uniform(-5, 5, shape).astype(npdt)
        rg = float(x.max() - x.min())
        h = mg.GridHierarchy.create(shape)
        L = h.num_levels()
        for stop in sorted({0, L - 1}):
            mc = mg.decompose_nonuniform(torch.from_numpy(x).cuda(), h, coords, stop, ws)
            want = o.decompose_nu(x, coords, stop)
            err = float(np.max(np.abs(mc.buffer.cpu().numpy().astype(np.float64) - want)))
            assert err <= tol * rg, (shape, stop, err / rg)
            back = mg.recompose_nonuniform(mc, coords, ws).cpu().numpy()
            assert float(np.max(np.abs(back.astype(np.float64) - x))) <= (1e-9 if dtype == "f64" else 1e-4) * rg
        eq = [np.linspace(0.0, 1.0, n) for n in shape]
        a = mg.decompose_nonuniform(torch.from_numpy(x).cuda(), h, eq, 0, ws).buffer.cpu().numpy()
        b = mg.decompose(torch.from_numpy(x).cuda(), h, 0, ws).buffer.cpu().numpy()
        assert float(np.max(np.abs(a.astype(np.float64) - b))) <= (1e-13 if dtype == "f64" else 1e-5) * rg, shape
