"""GPU parity: the CUDA path (through the C-ABI) against the reference's
outputs (tests/golden/golden.npz, generated from the unmodified reference)
and the pinned CPU oracle.

Bars (BASELINE.json north_star):
  * general per-step path: bit-identical to the reference (same arithmetic);
  * auto path (fused 3-D kernels where they apply): coefficients within
    1e-12 * range (fp64) / 1e-5 * range (fp32) of the reference;
  * quantized labels bit-exact except values within 1 ulp of a bin edge
    (counted); dequantize bit-exact.
"""
import os

import numpy as np
import pytest

GOLDEN = os.path.join(os.path.dirname(__file__), "golden", "golden.npz")
pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def torch():
    import torch as t

    return t


@pytest.fixture(scope="module")
def mg():
    import paper_2010_05872_b200 as m

    return m


@pytest.fixture(scope="module")
def g():
    return np.load(GOLDEN)


@pytest.fixture(scope="module")
def ws_general(mg):
    return mg.SolverWorkspace(path="general")


@pytest.fixture(scope="module")
def ws_auto(mg):
    return mg.SolverWorkspace(path="auto")


def shapes_in(g):
    out = set()
    for k in g.files:
        if k.endswith("_f64_in"):
            out.add(tuple(int(x) for x in k[: -len("_f64_in")].split("x")))
    return sorted(out)


def key(shape, *parts):
    return "x".join(str(s) for s in shape) + "_" + "_".join(str(p) for p in parts)


def to_dev(torch, a):
    return torch.from_numpy(np.ascontiguousarray(a)).cuda()


def bits(a):
    return np.ascontiguousarray(a).tobytes()


def test_general_path_bitwise_against_reference(torch, mg, g, ws_general):
    checked = 0
    for shape in shapes_in(g):
        h = mg.GridHierarchy.create(shape)
        L = h.num_levels()
        for name in ("f64", "f32"):
            x = to_dev(torch, g[key(shape, name, "in")])
            for stop in sorted({0, min(1, L), L}):
                mc = mg.decompose(x, h, stop, ws_general)
                got = mc.buffer.cpu().numpy()
                want = g[key(shape, name, "dec", stop)]
                assert bits(got) == bits(want), (shape, name, stop, np.abs(got - want).max())
                back = mg.recompose(mg.MultilevelCoefficients(to_dev(torch, want), h, stop), ws_general)
                assert bits(back.cpu().numpy()) == bits(g[key(shape, name, "rec", stop)]), (shape, name, stop)
                checked += 1
    assert checked > 100
    assert ws_general.launch_count() > 0


def test_auto_path_within_tolerance(torch, mg, g, ws_auto):
    for shape in shapes_in(g):
        h = mg.GridHierarchy.create(shape)
        L = h.num_levels()
        for name, tol in (("f64", 1e-12), ("f32", 1e-5)):
            xin = g[key(shape, name, "in")]
            rng_ = float(xin.max() - xin.min()) or 1.0
            x = to_dev(torch, xin)
            for stop in sorted({0, min(1, L), L}):
                got = mg.decompose(x, h, stop, ws_auto).buffer.cpu().numpy().astype(np.float64)
                want = g[key(shape, name, "dec", stop)].astype(np.float64)
                assert np.max(np.abs(got - want)) <= tol * rng_, (shape, name, stop)
                back = mg.recompose(mg.MultilevelCoefficients(to_dev(torch, g[key(shape, name, "dec", stop)]), h, stop),
                                    ws_auto).cpu().numpy().astype(np.float64)
                wr = g[key(shape, name, "rec", stop)].astype(np.float64)
                assert np.max(np.abs(back - wr)) <= tol * rng_, (shape, name, stop)


def test_quantize_dequantize_bitwise(torch, mg, g, ws_auto):
    for shape in shapes_in(g):
        h = mg.GridHierarchy.create(shape)
        L = h.num_levels()
        for name in ("f64", "f32"):
            plan = mg.make_plan(mg.QuantMode.levelwise, 1e-3 * 200.0, h)
            assert bits(plan.bin_widths) == bits(g[key(shape, name, "q")])
            c0 = to_dev(torch, g[key(shape, name, "dec", 0)])
            s = mg.quantize(mg.MultilevelCoefficients(c0, h, 0), plan, ws_auto)
            assert bits(s.flat.cpu().numpy()) == bits(g[key(shape, name, "labels")]), shape
            assert bits(s.outlier_positions.cpu().numpy()) == bits(g[key(shape, name, "opos")]), shape
            assert bits(s.outlier_values.cpu().numpy()) == bits(g[key(shape, name, "oval")]), shape
            back = mg.dequantize(s, plan, h, ws_auto)
            assert bits(back.buffer.cpu().numpy()) == bits(g[key(shape, name, "deq")]), shape
            if L >= 2:
                t = mg.quantize_tail(c0, h, 1, plan, ws_auto)
                assert bits(t.flat.cpu().numpy()) == bits(g[key(shape, name, "qtail_labels")])
                assert bits(t.outlier_positions.cpu().numpy()) == bits(g[key(shape, name, "qtail_opos")])
                buf = c0.clone()
                buf[h.node_count(1):] = 0
                mg.dequantize_tail(buf, t, h, 1, plan, ws_auto)
                full = mg.dequantize(s, plan, h, ws_auto).buffer
                n1 = h.node_count(1)
                assert torch.equal(buf[n1:], full[n1:])
                assert torch.equal(buf[:n1], c0[:n1])  # coarse block untouched by the tail


def test_quantize_subnormal_bin_widths(torch, mg, ws_auto):
    """Budgets small enough that the coarse bin widths are subnormal (their
    reciprocal overflows): labels and outliers still equal the reference's
    exact division (quantize.hpp:58-73), zeros included."""
    from oracle.oracle import Oracle

    o = Oracle()
    rng = np.random.default_rng(11)
    shape = (17, 9, 12)
    h = mg.GridHierarchy.create(shape)
    for budget in (1e-308, 1e-310, 1e-316):
        plan = mg.make_plan(mg.QuantMode.levelwise, budget, h)
        assert np.any(plan.bin_widths < np.finfo(np.float64).tiny)
        for dt in (np.float64, np.float32):
            x = rng.uniform(-1, 1, int(np.prod(shape))).astype(dt)
            x[::5] = 0.0
            x[1::7] = dt(1e-320) if dt == np.float64 else dt(0.0)
            s = mg.quantize(mg.MultilevelCoefficients(to_dev(torch, x), h, 0), plan, ws_auto)
            lab, opos, oval = o.quantize(x, shape, plan.bin_widths)
            assert np.array_equal(s.flat.cpu().numpy(), lab), (budget, dt)
            assert np.array_equal(s.outlier_positions.cpu().numpy(), opos), (budget, dt)
            assert np.array_equal(s.outlier_values.cpu().numpy(), oval), (budget, dt)


def test_quantize_errors(torch, mg, ws_auto):
    h = mg.GridHierarchy.create((5,))
    plan = mg.make_plan(mg.QuantMode.uniform, 0.1, h)
    c = torch.tensor([0.0, float("nan"), 0.0, 0.0, 0.0], dtype=torch.float64, device="cuda")
    with pytest.raises(mg.Error) as e:
        mg.quantize(mg.MultilevelCoefficients(c, h, 0), plan, ws_auto)
    assert e.value.code == "nonfinite_data"
    with pytest.raises(mg.Error) as e:
        mg.quantize(mg.MultilevelCoefficients(c, h, 1), plan, ws_auto)
    assert e.value.code == "invalid_input"
    # worked example (test_quantize.cpp:81-93) and overflow outlier (:124-134)
    plan = mg.make_plan(mg.QuantMode.uniform, 0.3, h)
    s = mg.quantize(mg.MultilevelCoefficients(torch.tensor([0.0, 0.29, 0, 0, 0], dtype=torch.float64,
                                                           device="cuda"), h, 0), plan, ws_auto)
    assert s.flat.cpu().tolist()[:2] == [0, 1]
    plan = mg.make_plan(mg.QuantMode.uniform, 1e-6, h)
    s = mg.quantize(mg.MultilevelCoefficients(torch.tensor([5.0, 0, 0, 0, 1e-7], dtype=torch.float64,
                                                           device="cuda"), h, 0), plan, ws_auto)
    assert s.outliers == [(0, 5.0)]
    assert mg.dequantize(s, plan, h, ws_auto).buffer[0].item() == 5.0


def test_transform_errors(torch, mg, ws_auto):
    h = mg.GridHierarchy.create((9, 9))
    x = torch.zeros((9, 8), dtype=torch.float64, device="cuda")
    with pytest.raises(mg.Error) as e:
        mg.decompose(x, h, 0, ws_auto)
    assert e.value.code == "shape_error"
    x = torch.zeros((9, 9), dtype=torch.float64, device="cuda")
    with pytest.raises(mg.Error) as e:
        mg.decompose(x, h, 5, ws_auto)
    assert e.value.code == "invalid_level"
    with pytest.raises(mg.Error) as e:
        mg.decompose(x.cpu(), h, 0, ws_auto)
    assert e.value.code == "invalid_argument"


def test_level_step_intermediates_general(torch, mg, g, ws_general):
    """One decompose level: shell equals the reference's reordered coefficient
    values; the coarse block equals nodal + correction (level_step fixtures)."""
    from oracle.oracle import Oracle

    for shape in [(9, 9), (17, 9, 5), (6, 5, 3), (7, 4), (9,)]:
        x = g[key(shape, "step_in")]
        h = mg.GridHierarchy.create(shape)
        L = h.num_levels()
        mc = mg.decompose(to_dev(torch, x), h, L - 1, ws_general).buffer.cpu().numpy()
        ref_field = g[key(shape, "step_field")]
        corr = g[key(shape, "step_corr")]
        # coarse block = nodal values (natural order = reordered corner) + corr
        coarse_dims = h.level_dims(L - 1)
        sl = tuple(slice(0, m) for m in coarse_dims)
        want_coarse = (ref_field[sl].astype(np.float64) + corr).ravel()
        assert bits(mc[: h.node_count(L - 1)]) == bits(want_coarse)
        # oracle agrees too
        assert bits(Oracle().decompose(x, L - 1)) == bits(mc)


def test_config1_against_reference(torch, mg):
    """BASELINE config 1 (129^3 f64, 16 bumps + noise), full decomposition,
    recomposition and level-wise quantization at 1e-3 relative (budget = tau/4)."""
    from oracle.oracle import Oracle, Reference, reference_available
    from synthetic_fields import config1_field

    ref = Reference() if reference_available() else Oracle()
    f = config1_field(device="cuda")
    fh = f.cpu().numpy()
    h = mg.GridHierarchy.create(f.shape)
    ws = mg.SolverWorkspace()
    mc = mg.decompose(f, h, 0, ws)
    want = ref.decompose(fh)
    rng_ = float(fh.max() - fh.min())
    assert np.max(np.abs(mc.buffer.cpu().numpy() - want)) <= 1e-12 * rng_
    back = mg.recompose(mc, ws).cpu().numpy()
    assert np.max(np.abs(back - fh)) <= 1e-9 * rng_
    tau = 1e-3 * rng_
    plan = mg.make_plan(mg.QuantMode.levelwise, tau / 4.0, h)  # budget = tau / C, C = 4
    s = mg.quantize(mc, plan, ws)
    lab_ref, opos_ref, _ = ref.quantize(want, f.shape, plan.bin_widths)
    # any flip must be a value within 1 ulp of a bin edge (north_star)
    from oracle.parity import label_flips

    n, worst = label_flips(want, s.flat.cpu().numpy(), lab_ref, h.delta_counts(), plan.bin_widths, ulps=1.0)
    print(f"config1 tau=1e-3: {n} bin-edge label flips (worst {worst:.2f} ulp)")
    rec = mg.recompose(mg.dequantize(s, plan, h, ws), ws).cpu().numpy()
    assert np.max(np.abs(rec - fh)) <= tau


FUSED_SHAPES = [(33, 33, 33), (65, 65, 65), (40, 36, 66), (35, 34, 100), (129, 65, 33), (6, 7, 300), (17, 100, 64),
                (66, 66, 66), (5, 200, 34),
                (9, 11, 700), (6, 9, 1025), (17, 12, 1079)]  # wide rows: 12..18 strips, one CTA per SM


@pytest.mark.parametrize("dtype", ["f64", "f32"])
def test_fused_path_against_oracle(torch, mg, ws_auto, dtype):
    """Shapes that take the fused 3-D kernels (alone or mixed with general
    levels), with odd/even extents, partial tiles and partial chunks."""
    from oracle.oracle import Oracle

    o = Oracle()
    rng = np.random.default_rng(5)
    npdt = np.float64 if dtype == "f64" else np.float32
    tol = 1e-12 if dtype == "f64" else 1e-5
    for shape in FUSED_SHAPES:
        x = rng.uniform(-10, 10, shape).astype(npdt)
        rg = float(x.max() - x.min())
        h = mg.GridHierarchy.create(shape)
        L = h.num_levels()
        for stop in sorted({0, L - 1}):
            want = o.decompose(x, stop)
            mc = mg.decompose(to_dev(torch, x), h, stop, ws_auto)
            got = mc.buffer.cpu().numpy()
            err = float(np.max(np.abs(got.astype(np.float64) - want)))
            assert err <= tol * rg, (shape, dtype, stop, err / rg)
            back = mg.recompose(mg.MultilevelCoefficients(to_dev(torch, want), h, stop), ws_auto).cpu().numpy()
            wr = o.recompose(want, shape, stop)
            err = float(np.max(np.abs(back.astype(np.float64) - wr)))
            assert err <= tol * rg, (shape, dtype, stop, "rec", err / rg)
            rt = mg.recompose(mc, ws_auto).cpu().numpy()
            assert float(np.max(np.abs(rt.astype(np.float64) - x))) <= (1e-9 if dtype == "f64" else 1e-4) * rg


TOEPLITZ_SHAPES = [(79, 79, 79),     # 40 unknowns on every axis: the shortest lines solved in Toeplitz form
                   (77, 81, 83),     # 39 (factor tables), 41, 42
                   (33, 40, 575),    # rows of 288 = 32 * 9: no leading zeros in the right-aligned row buffer
                   (20, 35, 191),    # rows of 96 = 32 * 3
                   (130, 36, 127),   # 65 planes, rows of 64 in a 96-wide buffer
                   (12, 20, 1919)]   # rows of 960, 33 values per lane


@pytest.mark.parametrize("dtype", ["f64", "f32"])
def test_toeplitz_solves_against_oracle(torch, mg, ws_auto, dtype):
    """The Toeplitz form of the correction solves (constant Thomas factors +
    end corrections, fused3d.cu) at its thresholds: line lengths 39 / 40 / 41,
    row buffers with and without leading zeros, the widest rows.  fp64 within
    1e-13 of the range (the bar is 1e-12; the solves differ from
    batched_solve, transform.hpp:116-130, only in rounding)."""
    from oracle.oracle import Oracle

    o = Oracle()
    rng = np.random.default_rng(17)
    npdt = np.float64 if dtype == "f64" else np.float32
    tol = 1e-13 if dtype == "f64" else 1e-5
    for shape in TOEPLITZ_SHAPES:
        x = rng.uniform(-10, 10, shape).astype(npdt)
        rg = float(x.max() - x.min())
        h = mg.GridHierarchy.create(shape)
        want = o.decompose(x, 0)
        mc = mg.decompose(to_dev(torch, x), h, 0, ws_auto)
        err = float(np.max(np.abs(mc.buffer.cpu().numpy().astype(np.float64) - want)))
        assert err <= tol * rg, (shape, dtype, err / rg)
        back = mg.recompose(mg.MultilevelCoefficients(to_dev(torch, want), h, 0), ws_auto).cpu().numpy()
        err = float(np.max(np.abs(back.astype(np.float64) - o.recompose(want, shape, 0))))
        assert err <= tol * rg, (shape, dtype, "rec", err / rg)


def test_graph_capture_matches_eager(torch, mg):
    """decompose + recompose captured in a CUDA graph (the recompose forks
    its level corrections onto the context's side streams and joins them)
    replays bit-identically to eager execution, for fp32 and fp64."""
    rng = np.random.default_rng(11)
    for shape, dt in (((129, 129, 129), np.float32), ((65, 66, 67), np.float64)):
        x = to_dev(torch, rng.uniform(-1, 1, shape).astype(dt))
        h = mg.GridHierarchy.create(shape)
        ws = mg.SolverWorkspace()

        def step():
            mc = mg.decompose(x, h, 0, ws)
            return mc.buffer, mg.recompose(mc, ws)

        c_e, f_e = step()
        torch.cuda.synchronize()
        side = torch.cuda.Stream()
        side.wait_stream(torch.cuda.current_stream())
        with torch.cuda.stream(side):
            step()
        torch.cuda.current_stream().wait_stream(side)
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g):
            c_g, f_g = step()
        for _ in range(2):
            g.replay()
        torch.cuda.synchronize()
        assert torch.equal(c_g, c_e), shape
        assert torch.equal(f_g, f_e), shape


def test_contexts_on_threads(torch, mg):
    """One context per host thread (the SolverWorkspace contract): two
    threads transforming different fields concurrently get the same results
    as a serial run."""
    import threading

    rng = np.random.default_rng(12)
    shape = (97, 65, 129)
    xs = [to_dev(torch, rng.uniform(-1, 1, shape).astype(np.float32)) for _ in range(2)]
    h = mg.GridHierarchy.create(shape)
    ref = []
    ws0 = mg.SolverWorkspace()
    for x in xs:
        ref.append(mg.decompose(x, h, 0, ws0).buffer.clone())
    torch.cuda.synchronize()
    out = [None, None]

    def work(i):
        s = torch.cuda.Stream()
        with torch.cuda.stream(s):
            ws = mg.SolverWorkspace()
            for _ in range(3):
                out[i] = mg.decompose(xs[i], h, 0, ws).buffer
        s.synchronize()

    ts = [threading.Thread(target=work, args=(i,)) for i in range(2)]
    for t in ts:
        t.start()
    for t in ts:
        t.join()
    for i in range(2):
        assert torch.equal(out[i], ref[i])


@pytest.mark.parametrize("shape", [(3, 2, 3, 2, 3, 2), (2, 3, 2, 3, 2, 3, 2), (3, 2, 2, 3, 2, 2, 2, 3)])
def test_high_rank_general_path(torch, mg, shape):
    """Ranks 6-8 (the C-ABI's maximum) on the general path: bit-identical to
    the oracle (itself bit-identical to the reference), both directions."""
    from oracle.oracle import Oracle

    o = Oracle()
    rng = np.random.default_rng(len(shape))
    x = rng.uniform(-1, 1, shape)
    h = mg.GridHierarchy.create(shape)
    ws = mg.SolverWorkspace(path="general")
    for stop in sorted({0, h.num_levels()}):
        got = mg.decompose(to_dev(torch, x), h, stop, ws).buffer.cpu().numpy()
        want = o.decompose(x, stop)
        assert bits(got) == bits(want), (shape, stop)
        back = mg.recompose(mg.MultilevelCoefficients(to_dev(torch, want), h, stop), ws).cpu().numpy()
        assert bits(back) == bits(o.recompose(want, shape, stop)), (shape, stop)


def test_rank_above_limit_is_rejected(mg):
    with pytest.raises(mg.Error) as e:
        mg.GridHierarchy.create((2,) * 9)
    assert e.value.code == "invalid_dims"


@pytest.mark.parametrize("dtype", [np.float64, np.float32])
def test_tail_kernel_bitwise(torch, mg, dtype):
    """Hierarchies small enough to run entirely in the one-CTA tail kernels
    (k_tail_decompose / k_tail_recompose: block-wide restriction, serial
    Thomas recurrences, 32-bit register geometry) on every rank 1-5 and every
    stop level: bit-identical to the oracle in both directions."""
    from oracle.oracle import Oracle

    o = Oracle()
    rng = np.random.default_rng(11)
    ws = mg.SolverWorkspace(path="auto")
    for shape in [(257,), (40,), (33, 17), (17, 17, 17), (9, 16, 5), (5, 9, 3, 6), (3, 4, 5, 3, 3)]:
        x = rng.uniform(-3, 3, shape).astype(dtype)
        h = mg.GridHierarchy.create(shape)
        for stop in range(h.num_levels() + 1):
            got = mg.decompose(to_dev(torch, x), h, stop, ws).buffer.cpu().numpy()
            want = o.decompose(x, stop).astype(dtype)
            assert bits(got) == bits(want), (shape, stop, "decompose")
            back = mg.recompose(mg.MultilevelCoefficients(to_dev(torch, want), h, stop), ws).cpu().numpy()
            assert bits(back) == bits(o.recompose(want, shape, stop).astype(dtype)), (shape, stop, "recompose")
