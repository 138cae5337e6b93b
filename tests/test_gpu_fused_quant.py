"""decompose_quantize / dequantize_recompose (the one-call forms of the ★
pairs of compress_field, pipeline.hpp:145-183, and decompress_field,
pipeline.hpp:235-260) against the two-call sequences: bit-identical
coefficients, labels, outliers and reconstruction, on the general path, the
fused 3-D path (where the finest shell is quantized under the rest of the
decomposition), with and without outliers, full and tail streams; and the
labels against the reference's golden labels."""
import os

import numpy as np
import pytest

pytestmark = pytest.mark.gpu
GOLDEN = os.path.join(os.path.dirname(__file__), "golden", "golden.npz")


@pytest.fixture(scope="module")
def torch():
    import torch as t

    return t


@pytest.fixture(scope="module")
def mg():
    import paper_2010_05872_b200 as m

    return m


def field(shape, dtype, seed):
    rng = np.random.default_rng(seed)
    ax = [np.linspace(0, 1, n) for n in shape]
    grids = np.meshgrid(*ax, indexing="ij")
    f = sum(np.sin((3 + i) * g + i) for i, g in enumerate(grids))
    f = f + 1e-3 * rng.standard_normal(shape)
    return np.ascontiguousarray(f.astype(dtype))


CASES = [
    ((65, 65, 65), np.float32, 0),
    ((129, 129, 129), np.float64, 0),
    ((100, 161, 97), np.float32, 0),
    ((129, 97, 161), np.float32, 2),
    ((257, 257), np.float64, 0),
    ((33, 17, 9, 9), np.float32, 1),
]


def same_stream(torch, a, b):
    assert torch.equal(a.flat, b.flat)
    assert torch.equal(a.outlier_positions, b.outlier_positions)
    assert torch.equal(a.outlier_values.view(torch.uint8), b.outlier_values.view(torch.uint8))


@pytest.mark.parametrize("shape,dtype,stop", CASES)
@pytest.mark.parametrize("rel", [1e-3, 1e-7])
def test_one_call_equals_two_calls(torch, mg, shape, dtype, stop, rel):
    x = field(shape, dtype, 7)
    d = torch.from_numpy(x).cuda()
    h = mg.GridHierarchy.create(shape)
    ws = mg.SolverWorkspace()
    rng_ = float(x.max() - x.min())
    plan = mg.make_plan(mg.QuantMode.levelwise, rel * rng_ / 4, h)  # 1e-7: labels beyond 16 bits -> outliers
    mc = mg.decompose(d, h, stop, ws)
    s = mg.quantize(mc, plan, ws) if stop == 0 else mg.quantize_tail(mc.buffer, h, stop, plan, ws)
    mc1, s1 = mg.decompose_quantize(d, h, plan, stop, ws)
    assert torch.equal(mc.buffer.view(torch.uint8), mc1.buffer.view(torch.uint8))
    same_stream(torch, s, s1)
    if rel < 1e-6:
        assert s.outlier_positions.numel() > 0
    # decompress side
    if stop == 0:
        back = mg.recompose(mg.dequantize(s, plan, h, ws), ws)
        back1 = mg.dequantize_recompose(s1, plan, h, ws)
    else:
        buf = mc.buffer.clone()
        mg.dequantize_tail(buf, s, h, stop, plan, ws)
        back = mg.recompose(mg.MultilevelCoefficients(buf, h, stop), ws)
        buf1 = mc.buffer.clone()
        buf1[h.node_count(stop):] = 0
        back1 = mg.dequantize_recompose(s1, plan, h, ws, stop_level=stop, buffer=buf1)
    assert torch.equal(back.view(torch.uint8), back1.view(torch.uint8))
    err = float((back1.double() - d.double()).abs().max())
    assert err <= rel * rng_ * 1.0000001


def test_labels_against_reference_golden(torch, mg):
    g = np.load(GOLDEN)
    shapes = sorted({tuple(int(v) for v in k[: -len("_f64_in")].split("x")) for k in g.files if k.endswith("_f64_in")})
    ws = mg.SolverWorkspace(path="general")  # bit-identical coefficients -> the reference's labels exactly
    for shape in shapes:
        h = mg.GridHierarchy.create(shape)
        for name in ("f64", "f32"):
            k = "x".join(str(s) for s in shape) + "_" + name
            x = torch.from_numpy(np.ascontiguousarray(g[k + "_in"])).cuda()
            plan = mg.make_plan(mg.QuantMode.levelwise, 1e-3 * 200.0, h)
            mc, s = mg.decompose_quantize(x, h, plan, 0, ws)
            assert mc.buffer.cpu().numpy().tobytes() == g[k + "_dec_0"].tobytes(), shape
            assert s.flat.cpu().numpy().tobytes() == g[k + "_labels"].tobytes(), shape
            assert s.outlier_positions.cpu().numpy().tobytes() == g[k + "_opos"].tobytes(), shape
            back = mg.dequantize_recompose(s, plan, h, ws)
            ref = mg.recompose(mg.dequantize(s, plan, h, ws), ws)
            assert torch.equal(back.view(torch.uint8), ref.view(torch.uint8))


def test_nonfinite_is_reported(torch, mg):
    x = field((65, 65, 65), np.float32, 1)
    x[40, 3, 7] = np.nan
    h = mg.GridHierarchy.create(x.shape)
    plan = mg.make_plan(mg.QuantMode.levelwise, 1e-3, h)
    with pytest.raises(mg.Error) as ei:
        mg.decompose_quantize(torch.from_numpy(x).cuda(), h, plan, 0, mg.SolverWorkspace())
    assert ei.value.code == "nonfinite_data"


def test_full_size_513(torch, mg):
    """Config 2 size: the one-call forms equal the two-call ones at 513^3 f32."""
    import synthetic_fields as sf

    d = sf.config2_field((513, 513, 513), seed=0, device="cuda").contiguous()
    h = mg.GridHierarchy.create(tuple(d.shape))
    ws = mg.SolverWorkspace()
    r = float(d.max() - d.min())
    plan = mg.make_plan(mg.QuantMode.levelwise, 1e-3 * r / 4, h)
    mc = mg.decompose(d, h, 0, ws)
    s = mg.quantize(mc, plan, ws)
    mc1, s1 = mg.decompose_quantize(d, h, plan, 0, ws)
    assert torch.equal(mc.buffer, mc1.buffer)
    same_stream(torch, s, s1)
    back1 = mg.dequantize_recompose(s1, plan, h, ws)
    back = mg.recompose(mg.dequantize(s, plan, h, ws), ws)
    assert torch.equal(back, back1)
    assert float((back1 - d).abs().max()) <= 1e-3 * r
