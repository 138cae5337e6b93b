"""Pins the CPU oracle (oracle/mgrx_oracle.c) before anything is checked
against it: bitwise against the reference's outputs committed in
tests/golden/golden.npz, against the reference tests' stated known answers,
and (when oracle/_ref is built) against the live reference on random shapes.
"""
import os

import numpy as np
import pytest

from oracle.oracle import Oracle, OracleError, Reference, reference_available

GOLDEN = os.path.join(os.path.dirname(__file__), "golden", "golden.npz")


@pytest.fixture(scope="module")
def g():
    return np.load(GOLDEN)


@pytest.fixture(scope="module")
def o():
    return Oracle()


def shapes_in(g):
    out = set()
    for k in g.files:
        if k.endswith("_f64_in"):
            out.add(tuple(int(x) for x in k[: -len("_f64_in")].split("x")))
    return sorted(out)


def k(shape, *parts):
    return "x".join(str(s) for s in shape) + "_" + "_".join(str(p) for p in parts)


def bits_equal(a, b):
    a = np.ascontiguousarray(a)
    b = np.ascontiguousarray(b)
    return a.shape == b.shape and a.dtype == b.dtype and a.tobytes() == b.tobytes()


def test_golden_decompose_recompose_bitwise(g, o):
    n = 0
    for shape in shapes_in(g):
        L = o.hierarchy(shape)[0]
        for name in ("f64", "f32"):
            x = g[k(shape, name, "in")]
            for stop in sorted({0, min(1, L), L}):
                c = o.decompose(x, stop)
                assert bits_equal(c, g[k(shape, name, "dec", stop)]), (shape, name, stop)
                r = o.recompose(g[k(shape, name, "dec", stop)], shape, stop)
                assert bits_equal(r, g[k(shape, name, "rec", stop)]), (shape, name, stop)
                n += 1
    assert n > 100


def test_golden_quantize_bitwise(g, o):
    for shape in shapes_in(g):
        L = o.hierarchy(shape)[0]
        for name, dt in (("f64", np.float64), ("f32", np.float32)):
            q = g[k(shape, name, "q")]
            assert bits_equal(o.make_plan(1, 1e-3 * 200.0, shape), q)
            c0 = g[k(shape, name, "dec", 0)]
            lab, opos, oval = o.quantize(c0, shape, q)
            assert bits_equal(lab, g[k(shape, name, "labels")])
            assert bits_equal(opos.astype(np.int64), g[k(shape, name, "opos")])
            assert bits_equal(oval, g[k(shape, name, "oval")])
            deq = o.dequantize(lab, opos, oval, shape, q, dtype=dt)
            assert bits_equal(deq, g[k(shape, name, "deq")])
            if L >= 2:
                lab, opos, _ = o.quantize(c0, shape, q, stop=1)
                assert bits_equal(lab, g[k(shape, name, "qtail_labels")])
                assert bits_equal(opos.astype(np.int64), g[k(shape, name, "qtail_opos")])


def test_golden_strided_reference_equivalence(g, o):
    # reference.hpp:237 == transform.hpp:509 bitwise (test_transform.cpp:396)
    for shape in [(17, 17), (9, 9, 9), (33, 5), (6, 9, 4)]:
        x = g[k(shape, "strided_in")]
        assert bits_equal(o.decompose(x), g[k(shape, "strided_dec")])


def test_known_answers(g, o):
    # test_transform.cpp:35-52
    assert np.array_equal(o.load_vector_1d([0, 0, 0, 0, 0]), [0, 0, 0])
    np.testing.assert_allclose(o.load_vector_1d([1, 1, 1, 1, 1]), [1, 2, 1], rtol=1e-15)
    np.testing.assert_allclose(o.load_vector_1d([0, 1, 0, 1, 0]), [0.5, 1, 0.5], rtol=1e-15)
    assert bits_equal(o.load_vector_1d([1, 1, 1, 1, 1]), g["ka_load_ones"])
    assert bits_equal(o.load_vector_1d([0, 1, 0, 1, 0]), g["ka_load_pure1d"])
    with pytest.raises(OracleError) as e:
        o.load_vector_1d([1, 2])
    assert e.value.errc == "degenerate_line"
    # test_transform.cpp:54-67 even-length boundary weights
    rng = np.random.default_rng(42)
    c = rng.uniform(-3, 3, 6)
    f = o.load_vector_1d(c)
    np.testing.assert_allclose(f[0], 5 / 12 * c[0] + 0.5 * c[1] + 1 / 12 * c[2], rtol=1e-15)
    np.testing.assert_allclose(f[2], 1 / 12 * c[2] + 0.5 * c[3] + 5 / 12 * c[4] + 0.5 * c[5], rtol=1e-15)
    # test_transform.cpp:103-137 constructed rhs, 2x2
    ones = o.solve_correction_1d([(2 / 3 if i in (0, 6) else 4 / 3) + (1 / 3 if i > 0 else 0) +
                                  (1 / 3 if i < 6 else 0) for i in range(7)])
    np.testing.assert_allclose(ones, 1.0, rtol=1e-14)
    assert bits_equal(ones, g["ka_solve_ones_rhs"])
    np.testing.assert_allclose(o.solve_correction_1d([1.0, 1.0]), [1.0, 1.0], rtol=1e-14)
    with pytest.raises(OracleError) as e:
        o.solve_correction_1d([1.0])
    assert e.value.errc == "degenerate_system"
    # test_reorder.cpp:192-199: 1D reorder clusters even indices first
    assert list(o.decompose(np.array([10.0, 11, 12, 13, 14]), stop=1) * 0 + 0) == [0] * 5  # shape sanity
    # test_grid.cpp
    L, ld, dc = o.hierarchy((65, 65, 65), 4)
    assert [int(np.prod(d)) for d in ld] == [125, 729, 4913, 35937, 274625]
    assert dc[4] == 238688 and np.array_equal(np.array(dc, dtype=np.uint64), g["ka_grid_65_4"])
    assert o.hierarchy((100, 500, 500))[0] == 6 == int(g["ka_levels_100x500x500"][0])
    assert o.hierarchy((2,))[0] == 0 and o.hierarchy((3, 1025))[0] == 1
    assert o.hierarchy((5,))[2] == [2, 1, 2]
    for bad, code in [((1, 5), "invalid_dims")]:
        with pytest.raises(OracleError) as e:
            o.hierarchy(bad)
        assert e.value.errc == code
    with pytest.raises(OracleError) as e:
        o.hierarchy((5, 5), 3)
    assert e.value.errc == "depth_exceeded"
    # test_quantize.cpp:19-43
    lw = o.make_plan(1, 0.125, (65, 65, 65), 4)
    np.testing.assert_allclose(lw[4] / lw[0], 238688.0 / 125.0, rtol=1e-12)
    assert bits_equal(lw, g["ka_plan_lw_65_4"])
    uni = o.make_plan(0, 0.125, (65, 65, 65), 4)
    np.testing.assert_allclose(uni, 2 * 0.125 / 5, rtol=1e-15)
    for p in (lw, uni):
        np.testing.assert_allclose(np.sum(p / 2), 0.125, rtol=1e-15)
    for bad in (0.0, -1.0):
        with pytest.raises(OracleError) as e:
            o.make_plan(0, bad, (65, 65, 65), 4)
        assert e.value.errc == "invalid_budget"
    # test_quantize.cpp:81-93 worked bin example
    q = o.make_plan(0, 0.3, (5,))
    np.testing.assert_allclose(q[0], 0.2, rtol=1e-15)
    lab, opos, oval = o.quantize(np.array([0.0, 0.29, 0, 0, 0]), (5,), q)
    assert lab[0] == 0 and lab[1] == 1 and len(opos) == 0
    # :124-134 alphabet overflow -> lossless outlier
    q = o.make_plan(0, 1e-6, (5,))
    lab, opos, oval = o.quantize(np.array([5.0, 0, 0, 0, 1e-7]), (5,), q)
    assert list(opos) == [0] and oval[0] == 5.0
    assert o.dequantize(lab, opos, oval, (5,), q)[0] == 5.0
    # :136-142 NaN refusal
    with pytest.raises(OracleError) as e:
        o.quantize(np.array([0.0, np.nan, 0, 0, 0]), (5,), o.make_plan(0, 0.1, (5,)))
    assert e.value.errc == "nonfinite_data"


@pytest.mark.skipif(not reference_available(), reason="oracle/_ref not built")
def test_oracle_matches_live_reference_random_shapes(o):
    r = Reference()
    rng = np.random.default_rng(77)
    for trial in range(40):
        d = int(rng.integers(1, 5))
        shape = tuple(int(rng.integers(2, 24 if d < 3 else 11)) for _ in range(d))
        dt = np.float32 if trial % 2 else np.float64
        x = rng.uniform(-50, 50, shape).astype(dt)
        L = r.hierarchy(shape)[0]
        for stop in sorted({0, L // 2, L}):
            a, b = o.decompose(x, stop), r.decompose(x, stop)
            assert bits_equal(a, b), (shape, stop)
            assert bits_equal(o.recompose(a, shape, stop), r.recompose(b, shape, stop)), (shape, stop)


def test_oracle_multilinear_fields_vanish(o):
    # test_transform.cpp:156-182
    for dims in [(9, 9), (5, 5, 5), (17, 9, 5)]:
        idx = np.indices(dims)
        f = 4.5 + sum((1.5 + i) * idx[i] for i in range(len(dims))).astype(np.float64)
        c = o.decompose(f)
        coarse = int(np.prod(o.hierarchy(dims)[1][0]))
        assert np.max(np.abs(c[coarse:])) <= 1e-9
