"""Adaptive stop decision on the GPU: choose_stop
(adaptive.hpp:99-104) over a level block in device memory must give the
reference's totals bit for bit (the per-block sums use the reference's
operation order; the blocks are summed in anchor order), hence the same
decision, for the sampled (step 8) and full (step 2) variants."""
import numpy as np
import pytest

from oracle.oracle import Reference


@pytest.fixture(scope="module")
def ref():
    return Reference()


def _block(shape, dtype, seed, smooth):
    rng = np.random.default_rng(seed)
    axes = np.meshgrid(*[np.linspace(0, 1, n) for n in shape], indexing="ij")
    x = sum(np.sin((2 + i) * np.pi * a + i) for i, a in enumerate(axes)) * smooth
    return (x + rng.normal(0, 1e-2, shape)).astype(dtype)


def test_reference_choose_stop_binding(ref):
    b = _block((17, 17, 17), np.float64, 0, 1.0)
    stop, lz, ip = ref.choose_stop(b, 1e-3, (0.518, 0.366, 0.259), 1.22)
    assert lz > 0 and ip > 0 and stop == (lz < ip)
    stop, lz, ip = ref.choose_stop(np.zeros((2, 5, 5)), 1e-3, (0.5, 0.3, 0.2), 1.2)
    assert stop and lz == 0 and ip == 0  # too small to sample


@pytest.mark.gpu
@pytest.mark.parametrize("shape,dtype", [((33, 33, 33), np.float32), ((65, 40, 17), np.float64), ((129, 129), np.float32),
                                         ((9, 11, 7, 13), np.float64), ((3, 3, 3), np.float32), ((2, 9, 9), np.float64),
                                         ((257, 257, 257), np.float32)])
@pytest.mark.parametrize("step", [8, 2])
@pytest.mark.parametrize("smooth", [1.0, 0.0])
def test_gpu_choose_stop_matches_reference(ref, shape, dtype, step, smooth):
    import torch

    import paper_2010_05872_b200 as mg

    if shape == (257, 257, 257) and step == 2:
        pytest.skip("full enumeration of 257^3 is slow on the CPU reference")
    b = _block(shape, dtype, 1, smooth)
    d = len(shape)
    pen = (0.518, 0.366, 0.259, 0.183)[:d]
    model = mg.PenaltyModel(lorenzo=1.22, interp=pen)
    for e in (1e-4, 1e-2):
        want = ref.choose_stop(b, e, pen, 1.22, step)
        got = mg.choose_stop(torch.from_numpy(b).cuda(), e, model, step, return_totals=True)
        assert got[1] == want[1] and got[2] == want[2], (got, want)
        assert got[0] == want[0]
