"""Out-of-bounds and coverage checks of the GPU passes through the C-ABI
(compute-sanitizer is not available on the B200 pool, so this is the
memory-safety net): every device buffer the library writes sits between
guard zones filled with a sentinel bit pattern, and the outputs start as
the sentinel.  After decompose / recompose / quantize / dequantize

* the guard zones are bit-for-bit unchanged (no write outside the buffer),
* no output element still holds the sentinel (every element is written),
* the results equal the unguarded call's (reads stayed in bounds too: the
  inputs' guard zones hold NaNs, which would poison any value read from them).

Shapes cover the fused 3-D passes (2- and 3-CTA variants, wide rows), the
general per-step path (2-D, 4-D), the tail kernel and partial stop levels.
"""
import ctypes as C

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

GUARD = 4096  # elements on each side
SHAPES = [((65, 65, 65), "f32"), ((129, 65, 33), "f32"), ((33, 40, 70), "f64"), ((17, 12, 1079), "f32"),
          ((9, 11, 700), "f64"), ((17, 12), "f64"), ((33, 20), "f32"), ((9, 8, 7, 6), "f32"), ((5, 5, 5), "f64")]


@pytest.fixture(scope="module")
def torch():
    import torch as t

    return t


@pytest.fixture(scope="module")
def mg():
    import paper_2010_05872_b200 as m

    return m


def _sentinel(torch, dtype):
    """A quiet NaN with a distinctive payload (fill_ keeps quiet NaN bits)."""
    if dtype == torch.float32:
        return torch.tensor([0x7FC0BAD1], dtype=torch.int32).view(torch.float32)[0]
    return torch.tensor([0x7FF8BADBADBADBAD], dtype=torch.int64).view(torch.float64)[0]


def _guarded(torch, n, dtype, fill):
    buf = torch.empty(n + 2 * GUARD, dtype=dtype, device="cuda")
    buf.fill_(fill)
    return buf, buf[GUARD:GUARD + n]


def _bits(torch, t):
    return t.view(torch.int32 if t.element_size() == 4 else torch.int64)


def _check_guards(torch, buf, n, sent):
    g = torch.cat([buf[:GUARD], buf[GUARD + n:]])
    s = _bits(torch, sent.reshape(1).to(buf.device)).expand(g.numel())
    assert torch.equal(_bits(torch, g), s), "write outside the buffer"


def _no_sentinel(torch, view, sent):
    s = _bits(torch, sent.reshape(1).to(view.device))
    assert not bool((_bits(torch, view) == s).any()), "output element left unwritten"


@pytest.mark.parametrize("shape,dt", SHAPES)
def test_guard_zones_and_coverage(torch, mg, shape, dt):
    from paper_2010_05872_b200._lib import lib

    dtype = torch.float32 if dt == "f32" else torch.float64
    code = 0 if dt == "f32" else 1
    sent = _sentinel(torch, dtype)
    rng = np.random.default_rng(7)
    n = int(np.prod(shape))
    x = torch.from_numpy(rng.uniform(-3, 3, n)).to(dtype).cuda()
    h = mg.GridHierarchy.create(shape)
    L = h.num_levels()
    ws = mg.SolverWorkspace()
    dims = (C.c_uint64 * len(shape))(*shape)
    for stop in sorted({0, 1, L - 1} & set(range(L + 1))):
        # decompose: NaN-guarded input, sentinel-filled guarded output
        xin_buf, xin = _guarded(torch, n, dtype, float("nan"))
        xin.copy_(x)
        out_buf, out = _guarded(torch, n, dtype, sent)
        ws._bind_stream()
        rc = lib.mgrx_gpu_decompose(ws.handle, code, len(shape), dims, L, stop, C.c_void_p(xin.data_ptr()),
                                    C.c_void_p(out.data_ptr()))
        assert rc == 0, rc
        torch.cuda.synchronize()
        _check_guards(torch, out_buf, n, sent)
        _no_sentinel(torch, out, sent)
        ref = mg.decompose(x.reshape(shape), h, stop, ws).buffer
        assert torch.equal(out, ref), (shape, stop)
        # recompose: NaN-guarded coefficients, sentinel-filled guarded field
        cin_buf, cin = _guarded(torch, n, dtype, float("nan"))
        cin.copy_(ref)
        back_buf, back = _guarded(torch, n, dtype, sent)
        ws._bind_stream()
        rc = lib.mgrx_gpu_recompose(ws.handle, code, len(shape), dims, L, stop, C.c_void_p(cin.data_ptr()),
                                    C.c_void_p(back.data_ptr()))
        assert rc == 0, rc
        torch.cuda.synchronize()
        _check_guards(torch, back_buf, n, sent)
        _no_sentinel(torch, back, sent)
        assert torch.equal(back, mg.recompose(mg.MultilevelCoefficients(ref, h, stop), ws).reshape(-1))
    # quantize / dequantize of a full decomposition
    coeffs = mg.decompose(x.reshape(shape), h, 0, ws).buffer
    plan = mg.make_plan(mg.QuantMode.levelwise, 1e-4, h)
    q = np.ascontiguousarray(plan.bin_widths, dtype=np.float64)
    lab_buf = torch.full((n + 2 * GUARD,), 0x7BADBAD, dtype=torch.int32, device="cuda")
    lab = lab_buf[GUARD:GUARD + n]
    cap = n
    pos_buf = torch.full((cap + 2 * GUARD,), -7, dtype=torch.int64, device="cuda")
    val_buf, _ = _guarded(torch, cap, dtype, sent)
    pos, val = pos_buf[GUARD:GUARD + cap], val_buf[GUARD:GUARD + cap]
    nout = C.c_uint64()
    ws._bind_stream()
    rc = lib.mgrx_gpu_quantize(ws.handle, code, len(shape), dims, L, 0, q.ctypes.data_as(C.POINTER(C.c_double)),
                               C.c_void_p(coeffs.data_ptr()), C.c_void_p(lab.data_ptr()), C.c_void_p(pos.data_ptr()),
                               C.c_void_p(val.data_ptr()), C.c_uint64(cap), C.byref(nout))
    assert rc == 0, rc
    torch.cuda.synchronize()
    k = int(nout.value)
    assert torch.equal(torch.cat([lab_buf[:GUARD], lab_buf[GUARD + n:]]),
                       torch.full((2 * GUARD,), 0x7BADBAD, dtype=torch.int32, device="cuda"))
    assert not bool((lab == 0x7BADBAD).any())
    assert bool((pos_buf[:GUARD] == -7).all()) and bool((pos_buf[GUARD + k:] == -7).all())
    _check_guards(torch, val_buf, cap, sent)
    s = mg.quantize(mg.MultilevelCoefficients(coeffs, h, 0), plan, ws)
    assert torch.equal(lab, s.flat) and k == s.outlier_positions.numel()
    assert torch.equal(pos[:k], s.outlier_positions)
    deq_buf, deq = _guarded(torch, n, dtype, sent)
    ws._bind_stream()
    rc = lib.mgrx_gpu_dequantize(ws.handle, code, len(shape), dims, L, 0, q.ctypes.data_as(C.POINTER(C.c_double)),
                                 C.c_void_p(lab.data_ptr()), C.c_void_p(pos.data_ptr()), C.c_void_p(val.data_ptr()),
                                 C.c_uint64(k), C.c_void_p(deq.data_ptr()))
    assert rc == 0, rc
    torch.cuda.synchronize()
    _check_guards(torch, deq_buf, n, sent)
    _no_sentinel(torch, deq, sent)
    assert torch.equal(deq, mg.dequantize(s, plan, h, ws).buffer)
