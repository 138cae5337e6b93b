"""GPU parity of the second-generation fused 3-D passes (csrc/fused_p2.cu):
fp32 levels with odd extents, (m2 - 1) % 32 == 0 and (m1 - 1) % 8 == 0 run
the plane pass (coefficients + load vector + axis-2 solve + chunk-local
axis-0 forward elimination, axis-1 solve by the last CTA of each plane), the
carry kernel and the column pass.  Checked against the pinned CPU oracle
(coefficients and recompose <= 1e-5 * range, the fp32 bar of north_star) on
shapes that cover one or many chunks and row tiles, chunk sizes 1..16 and
levels mixed with the other paths.
"""
import os

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

P2_SHAPES = [(65, 65, 65), (129, 129, 129), (17, 65, 129), (257, 65, 65), (41, 65, 65), (33, 257, 65),
             (21, 9, 65), (9, 65, 513)]


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


def _ws(mg, chunk=None, p2=True):
    """A workspace whose plans are built under the given p2 settings (the
    environment is read when a plan is first built)."""
    old = {k: os.environ.get(k) for k in ("MGRX_P2_CHUNK", "MGRX_P2")}
    try:
        if chunk is None:
            os.environ.pop("MGRX_P2_CHUNK", None)
        else:
            os.environ["MGRX_P2_CHUNK"] = str(chunk)
        os.environ["MGRX_P2"] = "1" if p2 else "0"
        ws = mg.SolverWorkspace()
        return ws, old
    except Exception:
        raise


def _restore(old):
    for k, v in old.items():
        if v is None:
            os.environ.pop(k, None)
        else:
            os.environ[k] = v


def _check(torch, mg, o, x, ws, stop=0):
    rg = float(x.max() - x.min())
    h = mg.GridHierarchy.create(x.shape)
    want = o.decompose(x, stop)
    mc = mg.decompose(torch.from_numpy(x).cuda(), h, stop, ws)
    got = mc.buffer.cpu().numpy()
    err = float(np.max(np.abs(got.astype(np.float64) - want)))
    assert err <= 1e-5 * rg, ("decompose", x.shape, err / rg)
    back = mg.recompose(mg.MultilevelCoefficients(torch.from_numpy(want.astype(np.float32)).cuda(), h, stop),
                        ws).cpu().numpy()
    wr = o.recompose(want.astype(np.float32), x.shape, stop)
    err = float(np.max(np.abs(back.astype(np.float64) - wr)))
    assert err <= 1e-5 * rg, ("recompose", x.shape, err / rg)
    rt = mg.recompose(mc, ws).cpu().numpy()
    assert float(np.max(np.abs(rt.astype(np.float64) - x))) <= 1e-4 * rg
    return got


@pytest.mark.parametrize("shape", P2_SHAPES)
def test_p2_against_oracle(torch, mg, o, shape):
    rng = np.random.default_rng(11)
    x = rng.uniform(-10, 10, shape).astype(np.float32)
    ws, old = _ws(mg)
    try:
        _check(torch, mg, o, x, ws)
        L = mg.GridHierarchy.create(shape).num_levels()
        _check(torch, mg, o, x, ws, stop=L - 2)
    finally:
        _restore(old)


@pytest.mark.parametrize("chunk", [1, 2, 3, 16])
def test_p2_chunk_sizes(torch, mg, o, chunk):
    rng = np.random.default_rng(12)
    x = rng.standard_normal((41, 49, 65)).astype(np.float32)
    ws, old = _ws(mg, chunk=chunk)
    try:
        _check(torch, mg, o, x, ws)
    finally:
        _restore(old)


def test_p2_matches_previous_fused_path(torch, mg):
    """The two fused implementations agree to rounding on a smooth field."""
    n = 129
    t = np.linspace(0, 1, n)
    x = (np.sin(7 * t)[:, None, None] * np.cos(5 * t)[None, :, None] * np.exp(t)[None, None, :]).astype(np.float32)
    h = mg.GridHierarchy.create(x.shape)
    ws_new, old = _ws(mg)
    _restore(old)
    ws_old, old = _ws(mg, p2=False)
    _restore(old)
    a = mg.decompose(torch.from_numpy(x).cuda(), h, 0, ws_new).buffer.cpu().numpy().astype(np.float64)
    b = mg.decompose(torch.from_numpy(x).cuda(), h, 0, ws_old).buffer.cpu().numpy().astype(np.float64)
    assert np.max(np.abs(a - b)) <= 1e-6 * float(x.max() - x.min())
