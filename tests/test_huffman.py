"""Label entropy coding on the GPU: encode_labels of
device-resident labels must produce the reference's byte stream
(src/huffman.cpp:209-255) exactly — same code lengths (heap order), same
canonical codes, same bit packing."""
import numpy as np
import pytest

from oracle.oracle import Reference


@pytest.fixture(scope="module")
def ref():
    return Reference()


def _labels(kind, n, seed):
    rng = np.random.default_rng(seed)
    if kind == "laplace":
        return np.rint(rng.laplace(0, 3, n)).astype(np.int32)
    if kind == "wide":
        return rng.integers(-60000, 60000, n).astype(np.int32)
    if kind == "single":
        return np.full(n, -7, np.int32)
    if kind == "two":
        return rng.choice(np.array([5, 9], np.int32), n, p=[0.9, 0.1])
    if kind == "skewed":  # long codes
        return np.minimum(rng.geometric(0.5, n), 45).astype(np.int32) - 20
    raise ValueError(kind)


def test_reference_encode_binding(ref):
    assert ref.encode_labels(np.zeros(0, np.int32)) == bytes(16)
    b = ref.encode_labels(np.array([1, 1, 2, 3], np.int32))
    assert b[:4] == (1).to_bytes(4, "little") and b[4:8] == (3).to_bytes(4, "little")


@pytest.mark.gpu
@pytest.mark.parametrize("kind", ["laplace", "wide", "single", "two", "skewed"])
@pytest.mark.parametrize("n", [1, 31, 4096, 4097, 100003, 3_000_001])
def test_gpu_encode_labels_matches_reference(ref, kind, n):
    import torch

    import paper_2010_05872_b200 as mg

    x = _labels(kind, n, n)
    want = ref.encode_labels(x)
    got = mg.encode_labels(torch.from_numpy(x).cuda())
    assert got == want


@pytest.mark.gpu
def test_gpu_encode_empty_and_alphabet_limit(ref):
    import torch

    import paper_2010_05872_b200 as mg

    assert mg.encode_labels(torch.zeros(0, dtype=torch.int32, device="cuda")) == bytes(16)
    with pytest.raises(mg.Error) as e:
        mg.encode_labels(torch.tensor([0, 1 << 17], dtype=torch.int32, device="cuda"))
    assert e.value.status == 15  # 1 + errc::invalid_input (label alphabet too large)


@pytest.mark.gpu
@pytest.mark.parametrize("dtype", ["float32", "float64"])
def test_gpu_field_stats(dtype):
    import torch

    import paper_2010_05872_b200 as mg

    x = torch.randn(1_000_003, dtype=getattr(torch, dtype), device="cuda")
    lo, hi, bad = mg.field_stats(x)
    assert lo == float(x.min()) and hi == float(x.max()) and bad == x.numel()
    x[777_777] = float("inf")
    x[900_001] = float("nan")
    lo2, hi2, bad2 = mg.field_stats(x)
    assert bad2 == 777_777 and lo2 == lo


@pytest.mark.gpu
@pytest.mark.parametrize("shape,dt", [((65, 65, 65), "f32"), ((129, 65, 33), "f32"), ((33, 40, 70), "f64"),
                                      ((9, 11, 700), "f32"), ((300, 258), "f64"), ((9, 8, 7, 6), "f32")])
def test_gpu_decompose_checked(shape, dt):
    """check_finite + range folded into the decompose's first plane pass
    (mgrx_gpu_decompose_checked; the fused 3-D shapes) or a separate pass
    (2-D / 4-D): the range equals the field's exact min / max, the output
    equals decompose's, and a NaN / inf raises the reference's
    nonfinite_data (MGRX_NONFINITE_DATA) with the first offset."""
    import ctypes as C

    import torch

    import paper_2010_05872_b200 as mg
    from paper_2010_05872_b200._lib import lib

    dtype = torch.float32 if dt == "f32" else torch.float64
    x = torch.randn(shape, dtype=dtype, device="cuda") * 3.0 + 1.0
    h = mg.GridHierarchy.create(shape)
    ws = mg.SolverWorkspace()
    out = torch.empty(x.numel(), dtype=dtype, device="cuda")
    dims = (C.c_uint64 * len(shape))(*shape)
    lo, hi, bad = C.c_double(), C.c_double(), C.c_uint64()
    code = 0 if dt == "f32" else 1
    ws._bind_stream()
    rc = lib.mgrx_gpu_decompose_checked(ws.handle, code, len(shape), dims, -1, 0, C.c_void_p(x.data_ptr()),
                                        C.c_void_p(out.data_ptr()), C.byref(lo), C.byref(hi), C.byref(bad))
    assert rc == 0, rc
    assert lo.value == float(x.min()) and hi.value == float(x.max()) and bad.value == x.numel()
    assert torch.equal(out, mg.decompose(x, h, 0, ws).buffer)
    y = x.clone().reshape(-1)
    y[y.numel() // 3] = float("nan")
    y[y.numel() // 2] = float("-inf")
    ws._bind_stream()
    rc = lib.mgrx_gpu_decompose_checked(ws.handle, code, len(shape), dims, -1, 0, C.c_void_p(y.data_ptr()),
                                        C.c_void_p(out.data_ptr()), C.byref(lo), C.byref(hi), C.byref(bad))
    assert rc == 9 and bad.value == y.numel() // 3, (rc, bad.value)  # MGRX_NONFINITE_DATA


@pytest.mark.gpu
@pytest.mark.parametrize("shape,dtype", [((33, 33, 33), np.float32), ((40, 17, 9), np.float64), ((129, 65), np.float32),
                                         ((9, 7, 11, 5), np.float64), ((1000,), np.float32)])
@pytest.mark.parametrize("e", [1e-1, 1e-4, 1e-9])
def test_gpu_lorenzo_matches_reference(ref, shape, dtype, e):
    """compress_lorenzo on the GPU (hyperplane wavefront): labels (as their
    encode_labels bytes) and outliers identical to the reference's; the
    tight bound forces outliers and the label-range cut-off."""
    import paper_2010_05872_b200 as mg

    rng = np.random.default_rng(len(shape))
    axes = np.meshgrid(*[np.linspace(0, 1, n) for n in shape], indexing="ij")
    x = (sum(np.sin(3 * a + i) for i, a in enumerate(axes)) + rng.normal(0, 1e-2, shape)).astype(dtype)
    labels, opos, oval = ref.lorenzo(x, e)
    enc, gpos, gval = mg.lorenzo_encode(x, e)
    assert enc == ref.encode_labels(labels)
    assert np.array_equal(gpos, opos) and np.array_equal(gval, oval)
