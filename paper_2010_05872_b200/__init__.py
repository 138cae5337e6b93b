"""B200-native multilevel decompose / recompose with level-wise quantization.

Python mirror of the reference's hot-path interface (namespace ``mgrx`` in
/root/reference/proj/core/include/mgrx): same names, argument meaning and
error behaviour, backed by the sm_100a kernels of ``libmgrx_b200.so``
through its C-ABI (include/mgrx_b200.h).  Device memory is torch CUDA
tensors; the work runs on the caller's current torch stream.

Reference interface                                  here
------------------------------------------------     -------------------------------
GridHierarchy::create (grid.hpp:30, grid.cpp:22)     GridHierarchy.create
SolverWorkspace (transform.hpp:48-75)                SolverWorkspace (GPU context)
decompose (transform.hpp:509)                        decompose
recompose (transform.hpp:517)                        recompose
make_plan (quantize.cpp:7)                           make_plan
quantize / quantize_tail (quantize.hpp:79,99)        quantize / quantize_tail
dequantize / dequantize_tail (quantize.hpp:118,137)  dequantize / dequantize_tail
mgrx::Error{errc} (error.hpp:27-36)                  Error(.code = errc name)

There is no CPU fallback: every transform call goes to the CUDA library and
raises if it is missing or no GPU is present.
"""
from __future__ import annotations

import ctypes as C
import enum
from dataclasses import dataclass, field as dc_field
from typing import List, Optional, Sequence

import numpy as np

from ._lib import LIB_PATH, lib, dp, u64p

__all__ = [
    "Error", "GridHierarchy", "SolverWorkspace", "MultilevelCoefficients", "QuantMode", "QuantizationPlan",
    "LabelStream", "decompose", "recompose", "decompose_nonuniform", "recompose_nonuniform", "make_plan",
    "quantize", "quantize_tail", "dequantize", "dequantize_tail", "decompose_quantize", "dequantize_recompose",
    "LIB_PATH",
]

ERRC = [
    "invalid_dims", "depth_exceeded", "invalid_level", "invalid_axis", "degenerate_line",
    "degenerate_system", "shape_error", "invalid_budget", "nonfinite_data", "decode_error",
    "not_an_artifact", "unsupported_version", "corrupt", "undefined_psnr", "invalid_input",
]
LOCAL = {100: "cuda_error", 101: "out_of_memory", 102: "invalid_argument", 103: "capacity_exceeded"}


class Error(RuntimeError):
    """mgrx::Error (error.hpp:27-36): ``code`` is the errc name."""

    def __init__(self, status: int, msg: str = ""):
        self.status = status
        self.code = ERRC[status - 1] if 1 <= status <= len(ERRC) else LOCAL.get(status, f"status_{status}")
        super().__init__(f"{self.code}: {msg}" if msg else self.code)


def _check(rc: int, ctx=None):
    if rc != 0:
        msg = lib.mgrx_gpu_last_error(ctx).decode() if ctx else ""
        raise Error(rc, msg)


def _dims_arr(dims: Sequence[int]):
    a = (C.c_uint64 * len(dims))(*[int(x) for x in dims])
    return a


# ------------------------------------------------------------------- grid

class GridHierarchy:
    """Decreasing sequence of subgrids (grid.hpp:13-76). Level 0 coarsest."""

    def __init__(self, dims, L, level_dims, deltas):
        self.dims = tuple(int(x) for x in dims)
        self._L = L
        self._level_dims = level_dims  # index = level
        self._deltas = deltas

    @staticmethod
    def create(dims: Sequence[int], levels: Optional[int] = None) -> "GridHierarchy":
        dims = [int(x) for x in dims]
        nd = len(dims)
        L = C.c_int()
        ld = (C.c_uint64 * (70 * max(nd, 1)))()
        dc = (C.c_uint64 * 70)()
        _check(lib.mgrx_hierarchy(nd, _dims_arr(dims) if nd else None, -1 if levels is None else int(levels),
                                  C.byref(L), ld, dc))
        n = L.value + 1
        level_dims = [tuple(int(ld[l * nd + i]) for i in range(nd)) for l in range(n)]
        return GridHierarchy(dims, L.value, level_dims, [int(dc[l]) for l in range(n)])

    @staticmethod
    def max_levels(dims: Sequence[int]) -> int:
        return GridHierarchy.create(dims).num_levels()

    def num_levels(self) -> int:
        return self._L

    def ndims(self) -> int:
        return len(self.dims)

    def _chk(self, level):
        if level < 0 or level > self._L:
            raise Error(3, f"level {level} out of range [0, {self._L}]")

    def level_dims(self, level: int):
        self._chk(level)
        return self._level_dims[level]

    def node_count(self, level: int) -> int:
        self._chk(level)
        return int(np.prod(self._level_dims[level]))

    def delta_count(self, level: int) -> int:
        self._chk(level)
        return self._deltas[level]

    def total_count(self) -> int:
        return self.node_count(self._L)

    def dims_per_level(self):
        """Finest first, like grid.hpp:73."""
        return list(reversed(self._level_dims))

    def delta_counts(self):
        return list(self._deltas)

    def __eq__(self, other):
        return isinstance(other, GridHierarchy) and self.dims == other.dims and self._L == other._L

    def __repr__(self):
        return f"GridHierarchy(dims={self.dims}, levels={self._L})"


# -------------------------------------------------------------- workspace

class SolverWorkspace:
    """GPU analogue of SolverWorkspace (transform.hpp:46-75): a context owning
    device scratch, uploaded per-level tables and cached launch plans on one
    device.  Not thread-safe; use one per host thread.  ``batch_size`` is
    accepted for signature compatibility (it is a CPU cache-blocking knob that
    cannot change results, test_transform.cpp:300)."""

    def __init__(self, batch_size: int = 32, device: Optional[int] = None, path: str = "auto"):
        import torch

        self.batch_size = batch_size
        self.device = torch.cuda.current_device() if device is None else int(device)
        self._torch = torch
        h = C.c_void_p()
        _check(lib.mgrx_gpu_ctx_create(self.device, C.byref(h)))
        self._h = h
        self.set_path(path)

    def set_path(self, path: str):
        _check(lib.mgrx_gpu_set_path(self._h, {"auto": 0, "general": 1}[path]), self._h)
        self.path = path

    def _bind_stream(self):
        s = self._torch.cuda.current_stream(self.device).cuda_stream
        _check(lib.mgrx_gpu_set_stream(self._h, C.c_void_p(s)), self._h)

    def prepare(self, hierarchy: "GridHierarchy"):  # SolverWorkspace::prepare (transform.hpp:58)
        return None

    def launch_count(self) -> int:
        return int(lib.mgrx_gpu_launch_count(self._h))

    def profile_begin(self):
        """Start per-kernel CUDA-event timing (mgrx_gpu_profile_begin)."""
        _check(lib.mgrx_gpu_profile_begin(self._h), self._h)

    def profile_end(self) -> dict:
        """{kernel tag: (total ms, launches)} since profile_begin."""
        cap = 64
        tags = C.create_string_buffer(32 * cap)
        ms = (C.c_double * cap)()
        cnt = (C.c_uint64 * cap)()
        n = C.c_int()
        _check(lib.mgrx_gpu_profile_end(self._h, tags, ms, cnt, cap, C.byref(n)), self._h)
        out = {}
        for i in range(min(n.value, cap)):
            name = tags.raw[32 * i: 32 * (i + 1)].split(b"\0", 1)[0].decode()
            out[name] = (float(ms[i]), int(cnt[i]))
        return out

    def synchronize(self):
        _check(lib.mgrx_gpu_synchronize(self._h), self._h)

    @property
    def handle(self):
        return self._h

    def close(self):
        if getattr(self, "_h", None) is not None and self._h.value:
            lib.mgrx_gpu_ctx_destroy(self._h)
            self._h = C.c_void_p()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


_default_ws: dict = {}


def _ws(ws):
    if ws is not None:
        return ws
    import torch

    dev = torch.cuda.current_device()
    if dev not in _default_ws:
        _default_ws[dev] = SolverWorkspace(device=dev)
    return _default_ws[dev]


# ------------------------------------------------------------- transform

def _dtype_code(t):
    import torch

    if t.dtype == torch.float32:
        return 0
    if t.dtype == torch.float64:
        return 1
    raise Error(102, f"unsupported dtype {t.dtype}")


def _require_cuda(t, what):
    if not t.is_cuda:
        raise Error(102, f"{what} must be a CUDA tensor")
    if not t.is_contiguous():
        raise Error(102, f"{what} must be contiguous")


@dataclass
class MultilevelCoefficients:
    """transform.hpp:158-163: level-centric buffer (coarse block, then each
    level's shell) + hierarchy + stop level.  ``buffer`` is a CUDA tensor."""

    buffer: "object"
    hierarchy: GridHierarchy
    stop_level: int = 0


def _levels_of(h: GridHierarchy) -> int:
    return h.num_levels()


def decompose(field, hierarchy: GridHierarchy, stop_level: int = 0,
              ws: Optional[SolverWorkspace] = None) -> MultilevelCoefficients:
    """decompose (transform.hpp:509-515). ``field`` is a CUDA tensor with the
    hierarchy's finest dims; it is not modified."""
    import torch

    ws = _ws(ws)
    _require_cuda(field, "field")
    if tuple(field.shape) != hierarchy.level_dims(hierarchy.num_levels()):
        raise Error(7, "field dims do not match hierarchy")
    if stop_level < 0 or stop_level > hierarchy.num_levels():
        raise Error(3, "stop level out of range")
    out = torch.empty(field.numel(), dtype=field.dtype, device=field.device)
    ws._bind_stream()
    d = _dims_arr(field.shape)
    _check(lib.mgrx_gpu_decompose(ws.handle, _dtype_code(field), field.dim(), d, _levels_of(hierarchy),
                                  int(stop_level), C.c_void_p(field.data_ptr()), C.c_void_p(out.data_ptr())),
           ws.handle)
    return MultilevelCoefficients(out, hierarchy, int(stop_level))


def recompose(coeffs: MultilevelCoefficients, ws: Optional[SolverWorkspace] = None):
    """recompose (transform.hpp:517-530) -> CUDA tensor of the finest dims."""
    import torch

    ws = _ws(ws)
    h = coeffs.hierarchy
    buf = coeffs.buffer
    _require_cuda(buf, "coeffs.buffer")
    if buf.numel() != h.total_count():
        raise Error(7, "buffer size != total node count")
    dims = h.level_dims(h.num_levels())
    out = torch.empty(dims, dtype=buf.dtype, device=buf.device)
    ws._bind_stream()
    _check(lib.mgrx_gpu_recompose(ws.handle, _dtype_code(buf), len(dims), _dims_arr(dims), h.num_levels(),
                                  int(coeffs.stop_level), C.c_void_p(buf.data_ptr()), C.c_void_p(out.data_ptr())),
           ws.handle)
    return out


def _coord_ptrs(coords, dims):
    if len(coords) != len(dims):
        raise Error(7, "one coordinate array per axis required")
    arrs = []
    for a, (c, n) in enumerate(zip(coords, dims)):
        c = np.ascontiguousarray(np.asarray(c, dtype=np.float64))
        if c.shape != (n,):
            raise Error(7, f"coords[{a}] must have {n} entries")
        arrs.append(c)
    ptrs = (dp * len(arrs))(*[a.ctypes.data_as(dp) for a in arrs])
    return arrs, ptrs


def decompose_nonuniform(field, hierarchy: GridHierarchy, coords, stop_level: int = 0,
                         ws: Optional[SolverWorkspace] = None) -> MultilevelCoefficients:
    """Nonuniform-coordinate decompose (no reference counterpart; equals
    ``decompose`` to rounding for equispaced coordinates)."""
    import torch

    ws = _ws(ws)
    _require_cuda(field, "field")
    if tuple(field.shape) != hierarchy.level_dims(hierarchy.num_levels()):
        raise Error(7, "field dims do not match hierarchy")
    keep, ptrs = _coord_ptrs(coords, field.shape)
    out = torch.empty(field.numel(), dtype=field.dtype, device=field.device)
    ws._bind_stream()
    _check(lib.mgrx_gpu_decompose_nonuniform(ws.handle, _dtype_code(field), field.dim(), _dims_arr(field.shape),
                                             hierarchy.num_levels(), int(stop_level), ptrs,
                                             C.c_void_p(field.data_ptr()), C.c_void_p(out.data_ptr())), ws.handle)
    return MultilevelCoefficients(out, hierarchy, int(stop_level))


def recompose_nonuniform(coeffs: MultilevelCoefficients, coords, ws: Optional[SolverWorkspace] = None):
    import torch

    ws = _ws(ws)
    h = coeffs.hierarchy
    buf = coeffs.buffer
    _require_cuda(buf, "coeffs.buffer")
    dims = h.level_dims(h.num_levels())
    keep, ptrs = _coord_ptrs(coords, dims)
    out = torch.empty(dims, dtype=buf.dtype, device=buf.device)
    ws._bind_stream()
    _check(lib.mgrx_gpu_recompose_nonuniform(ws.handle, _dtype_code(buf), len(dims), _dims_arr(dims),
                                             h.num_levels(), int(coeffs.stop_level), ptrs,
                                             C.c_void_p(buf.data_ptr()), C.c_void_p(out.data_ptr())), ws.handle)
    return out


# -------------------------------------------------------------- quantize

# ------------------------------------------------------ adaptive stop

@dataclass
class PenaltyModel:
    """adaptive.hpp:16-21 (the calibrated 3-D constants by default; other
    ranks take the reference's estimate_penalty_factors values)."""

    lorenzo: float = 1.22
    interp: tuple = (0.518, 0.366, 0.259)


def choose_stop(level_block, e: float, model: Optional[PenaltyModel] = None, anchor_step: int = 8,
                ws: Optional[SolverWorkspace] = None, return_totals: bool = False):
    """choose_stop (adaptive.hpp:99-104) on a level block in device memory
    (CUDA tensor, natural order): True = stop here (the Lorenzo estimate is
    lower).  anchor_step 2 is choose_stop_full.  The sampled blocks'
    estimates run on the GPU; the totals are bit-identical to the
    reference's."""
    ws = _ws(ws)
    model = model or PenaltyModel()
    _require_cuda(level_block, "level_block")
    d = level_block.dim()
    if len(model.interp) < d:
        raise Error(15, "penalty model rank too small")
    pen = (C.c_double * d)(*[float(x) for x in model.interp[:d]])
    tot = (C.c_double * 2)()
    stop = C.c_int(0)
    ws._bind_stream()
    _check(lib.mgrx_gpu_choose_stop(ws.handle, _dtype_code(level_block), d, _dims_arr(level_block.shape),
                                    C.c_void_p(level_block.data_ptr()), float(e), pen, float(model.lorenzo),
                                    int(anchor_step), tot, C.byref(stop)), ws.handle)
    if return_totals:
        return bool(stop.value), float(tot[0]), float(tot[1])
    return bool(stop.value)


def field_stats(field, ws: Optional[SolverWorkspace] = None):
    """check_finite (pipeline.hpp:113-118) + range in one device read:
    (min, max) of the finite values and the first non-finite offset (numel
    when all are finite)."""
    ws = _ws(ws)
    _require_cuda(field, "field")
    lo, hi, bad = C.c_double(0), C.c_double(0), C.c_uint64(0)
    ws._bind_stream()
    _check(lib.mgrx_gpu_field_stats(ws.handle, _dtype_code(field), field.numel(), C.c_void_p(field.data_ptr()),
                                    C.byref(lo), C.byref(hi), C.byref(bad)), ws.handle)
    return lo.value, hi.value, bad.value


def lorenzo_encode(block, e: float, ws: Optional[SolverWorkspace] = None):
    """compress_lorenzo (lorenzo.hpp:87-128) of a host numpy block on the GPU:
    (encode_labels bytes of the labels, outlier positions, outlier values)."""
    import numpy as np

    ws = _ws(ws)
    block = np.ascontiguousarray(block)
    code = {np.dtype(np.float32): 0, np.dtype(np.float64): 1}[block.dtype]
    n = block.size
    enc = np.empty(16 + (1 << 17) + 4 * n + 64, np.uint8)
    cap = max(n, 1)
    opos = np.empty(cap, np.uint64)
    oval = np.empty(cap, block.dtype)
    esz, nout = C.c_uint64(0), C.c_uint64(0)
    _check(lib.mgrx_host_lorenzo(ws.handle, code, block.ndim, _dims_arr(block.shape),
                                 block.ctypes.data_as(C.c_void_p), float(e), enc.ctypes.data_as(C.c_void_p),
                                 enc.size, C.byref(esz), opos.ctypes.data_as(C.POINTER(C.c_uint64)),
                                 oval.ctypes.data_as(C.c_void_p), cap, C.byref(nout)), ws.handle)
    return enc[:esz.value].tobytes(), opos[:nout.value], oval[:nout.value]


def encode_labels(labels, ws: Optional[SolverWorkspace] = None) -> bytes:
    """encode_labels (huffman.hpp:14): the reference's canonical-Huffman byte
    stream of an int32 CUDA tensor of labels, histogram and bit packing on
    the GPU (only the encoded bytes come to the host)."""
    import torch

    ws = _ws(ws)
    _require_cuda(labels, "labels")
    if labels.dtype != torch.int32:
        raise Error(102, "labels must be int32")
    n = labels.numel()
    size = C.c_uint64(0)
    cap = 16 + (1 << 17) + 4 * n + 64
    buf = (C.c_uint8 * cap)()
    ws._bind_stream()
    _check(lib.mgrx_gpu_encode_labels(ws.handle, C.c_void_p(labels.data_ptr()), n, buf, cap, C.byref(size)),
           ws.handle)
    return bytes(buf[:size.value])


class QuantMode(enum.IntEnum):  # quantize.hpp:14
    uniform = 0
    levelwise = 1


@dataclass
class QuantizationPlan:  # quantize.hpp:24-31
    mode: QuantMode = QuantMode.levelwise
    budget: float = 0.0
    bin_widths: np.ndarray = dc_field(default_factory=lambda: np.zeros(0))
    range: float = 0.0

    def num_levels(self) -> int:
        return len(self.bin_widths) - 1


def make_plan(mode: QuantMode, budget: float, hierarchy: GridHierarchy) -> QuantizationPlan:
    """make_plan (quantize.cpp:7-24)."""
    L = hierarchy.num_levels()
    q = (C.c_double * (L + 1))()
    dims = hierarchy.dims
    _check(lib.mgrx_make_plan(int(mode), C.c_double(budget), len(dims), _dims_arr(dims), L, q))
    return QuantizationPlan(QuantMode(int(mode)), float(budget), np.array(q[:], dtype=np.float64))


@dataclass
class LabelStream:
    """quantize.hpp:47-51.  ``labels`` is one CUDA int32 tensor per level
    (views into ``flat``); outliers are (positions uint64, values) tensors in
    strictly increasing position order."""

    flat: "object"
    labels: List["object"]
    outlier_positions: "object"
    outlier_values: "object"

    @property
    def outliers(self):
        return list(zip(self.outlier_positions.cpu().tolist(), self.outlier_values.cpu().tolist()))


def _quantize(buffer, h: GridHierarchy, stop: int, plan: QuantizationPlan, ws) -> LabelStream:
    import torch

    ws = _ws(ws)
    _require_cuda(buffer, "buffer")
    if plan.num_levels() != h.num_levels():
        raise Error(7, "plan does not match hierarchy")
    L = h.num_levels()
    first = 0 if stop == 0 else stop + 1
    base = 0 if stop == 0 else h.node_count(stop)
    nlab = h.total_count() - base
    flat = torch.empty(nlab, dtype=torch.int32, device=buffer.device)
    q = np.ascontiguousarray(plan.bin_widths, dtype=np.float64)
    n_out = C.c_uint64()
    dims = h.dims
    cap = max(1, min(nlab, max(1 << 16, nlab >> 8)))  # 0.4 % of the labels: a retry is rare
    ws._bind_stream()
    while True:
        opos = torch.empty(cap, dtype=torch.int64, device=buffer.device)
        oval = torch.empty(cap, dtype=buffer.dtype, device=buffer.device)
        rc = lib.mgrx_gpu_quantize(ws.handle, _dtype_code(buffer), len(dims), _dims_arr(dims), L, int(stop),
                                   q.ctypes.data_as(dp), C.c_void_p(buffer.data_ptr()), C.c_void_p(flat.data_ptr()),
                                   C.c_void_p(opos.data_ptr()), C.c_void_p(oval.data_ptr()), C.c_uint64(cap),
                                   C.byref(n_out))
        if rc == 103:  # capacity exceeded: retry with the exact count
            cap = int(n_out.value)
            continue
        _check(rc, ws.handle)
        break
    k = int(n_out.value)
    labels, pos = [], 0
    for l in range(first, L + 1):
        labels.append(flat[pos:pos + h.delta_count(l)])
        pos += h.delta_count(l)
    return LabelStream(flat, labels, opos[:k], oval[:k])


def quantize(coeffs: MultilevelCoefficients, plan: QuantizationPlan,
             ws: Optional[SolverWorkspace] = None) -> LabelStream:
    """quantize (quantize.hpp:79-95): requires a fully decomposed buffer."""
    if coeffs.stop_level != 0:
        raise Error(15, "quantize expects a fully decomposed buffer")
    return _quantize(coeffs.buffer, coeffs.hierarchy, 0, plan, ws)


def quantize_tail(buffer, hierarchy: GridHierarchy, stop_level: int, plan: QuantizationPlan,
                  ws: Optional[SolverWorkspace] = None) -> LabelStream:
    """quantize_tail (quantize.hpp:99-114): levels above stop_level only."""
    return _quantize(buffer, hierarchy, int(stop_level), plan, ws)


def decompose_quantize(field, hierarchy: GridHierarchy, plan: QuantizationPlan, stop_level: int = 0,
                       ws: Optional[SolverWorkspace] = None):
    """decompose (transform.hpp:485-506) + quantize / quantize_tail
    (quantize.hpp:79-114) as compress_field runs them (pipeline.hpp:145-183),
    in one call: the finest shell's labels are produced under the rest of the
    decomposition.  Returns (MultilevelCoefficients, LabelStream), identical to
    ``decompose`` followed by ``quantize`` / ``quantize_tail``."""
    import torch

    ws = _ws(ws)
    h = hierarchy
    _require_cuda(field, "field")
    if tuple(field.shape) != h.level_dims(h.num_levels()):
        raise Error(7, "field dims do not match hierarchy")
    if stop_level < 0 or stop_level > h.num_levels():
        raise Error(3, "stop level out of range")
    if plan.num_levels() != h.num_levels():
        raise Error(7, "plan does not match hierarchy")
    stop = int(stop_level)
    L = h.num_levels()
    first = 0 if stop == 0 else stop + 1
    base = 0 if stop == 0 else h.node_count(stop)
    nlab = h.total_count() - base
    out = torch.empty(field.numel(), dtype=field.dtype, device=field.device)
    flat = torch.empty(nlab, dtype=torch.int32, device=field.device)
    q = np.ascontiguousarray(plan.bin_widths, dtype=np.float64)
    n_out = C.c_uint64()
    cap = max(1, min(nlab, max(1 << 16, nlab >> 8)))
    opos = torch.empty(cap, dtype=torch.int64, device=field.device)
    oval = torch.empty(cap, dtype=field.dtype, device=field.device)
    ws._bind_stream()
    d = _dims_arr(field.shape)
    rc = lib.mgrx_gpu_decompose_quantize(ws.handle, _dtype_code(field), field.dim(), d, L, stop,
                                         C.c_void_p(field.data_ptr()), q.ctypes.data_as(dp),
                                         C.c_void_p(out.data_ptr()), C.c_void_p(flat.data_ptr()),
                                         C.c_void_p(opos.data_ptr()), C.c_void_p(oval.data_ptr()), C.c_uint64(cap),
                                         C.byref(n_out))
    mc = MultilevelCoefficients(out, h, stop)
    if rc == 103:  # capacity exceeded: the coefficients are complete, redo the quantizer with the exact count
        return mc, _quantize(out, h, stop, plan, ws)
    _check(rc, ws.handle)
    k = int(n_out.value)
    labels, pos = [], 0
    for l in range(first, L + 1):
        labels.append(flat[pos:pos + h.delta_count(l)])
        pos += h.delta_count(l)
    return mc, LabelStream(flat, labels, opos[:k], oval[:k])


def dequantize_recompose(stream: LabelStream, plan: QuantizationPlan, hierarchy: GridHierarchy,
                         ws: Optional[SolverWorkspace] = None, dtype=None, stop_level: int = 0, buffer=None):
    """dequantize / dequantize_tail (quantize.hpp:118-150) + recompose
    (transform.hpp:509-530) as decompress_field runs them (pipeline.hpp:235-260),
    in one call.  For ``stop_level`` > 0 pass ``buffer`` holding the decoded
    coarse block (its shells are overwritten).  Returns the field."""
    import torch

    ws = _ws(ws)
    h = hierarchy
    stop = int(stop_level)
    L = h.num_levels()
    first = 0 if stop == 0 else stop + 1
    if len(stream.labels) != L + 1 - first:
        raise Error(7, "label stream does not match hierarchy")
    for l, lv in zip(range(first, L + 1), stream.labels):
        if lv.numel() != h.delta_count(l):
            raise Error(7, "label count mismatch")
    if stop > 0 and buffer is None:
        raise Error(15, "a tail stream needs the buffer holding the coarse block")
    dtype = dtype or (buffer.dtype if buffer is not None else stream.outlier_values.dtype)
    if buffer is None:
        buffer = torch.empty(h.total_count(), dtype=dtype, device=stream.flat.device)
    _require_cuda(buffer, "buffer")
    flat = stream.flat if stream.flat.numel() == sum(x.numel() for x in stream.labels) else torch.cat(stream.labels)
    q = np.ascontiguousarray(plan.bin_widths, dtype=np.float64)
    dims = h.level_dims(L)
    out = torch.empty(dims, dtype=buffer.dtype, device=buffer.device)
    n = int(stream.outlier_positions.numel())
    ws._bind_stream()
    _check(lib.mgrx_gpu_dequantize_recompose(ws.handle, _dtype_code(buffer), len(dims), _dims_arr(dims), L, stop,
                                             q.ctypes.data_as(dp), C.c_void_p(flat.data_ptr()),
                                             C.c_void_p(stream.outlier_positions.data_ptr() if n else 0),
                                             C.c_void_p(stream.outlier_values.data_ptr() if n else 0),
                                             C.c_uint64(n), C.c_void_p(buffer.data_ptr()),
                                             C.c_void_p(out.data_ptr())), ws.handle)
    return out


def _dequantize(stream: LabelStream, plan: QuantizationPlan, h: GridHierarchy, stop: int, out, ws):
    ws = _ws(ws)
    L = h.num_levels()
    first = 0 if stop == 0 else stop + 1
    if len(stream.labels) != L + 1 - first:
        raise Error(7, "label stream does not match hierarchy")
    for l, lv in zip(range(first, L + 1), stream.labels):
        if lv.numel() != h.delta_count(l):
            raise Error(7, "label count mismatch")
    import torch

    flat = stream.flat if stream.flat.numel() == sum(x.numel() for x in stream.labels) else torch.cat(stream.labels)
    q = np.ascontiguousarray(plan.bin_widths, dtype=np.float64)
    dims = h.dims
    n = int(stream.outlier_positions.numel())
    ws._bind_stream()
    _check(lib.mgrx_gpu_dequantize(ws.handle, _dtype_code(out), len(dims), _dims_arr(dims), L, int(stop),
                                   q.ctypes.data_as(dp), C.c_void_p(flat.data_ptr()),
                                   C.c_void_p(stream.outlier_positions.data_ptr() if n else 0),
                                   C.c_void_p(stream.outlier_values.data_ptr() if n else 0), C.c_uint64(n),
                                   C.c_void_p(out.data_ptr())), ws.handle)
    return out


def dequantize(stream: LabelStream, plan: QuantizationPlan, hierarchy: GridHierarchy,
               ws: Optional[SolverWorkspace] = None, dtype=None) -> MultilevelCoefficients:
    """dequantize (quantize.hpp:118-135)."""
    import torch

    dtype = dtype or stream.outlier_values.dtype
    # every position of a full decomposition carries a label: no zero fill
    out = torch.empty(hierarchy.total_count(), dtype=dtype, device=stream.flat.device)
    _dequantize(stream, plan, hierarchy, 0, out, ws)
    return MultilevelCoefficients(out, hierarchy, 0)


def dequantize_tail(buffer, stream: LabelStream, hierarchy: GridHierarchy, stop_level: int,
                    plan: QuantizationPlan, ws: Optional[SolverWorkspace] = None):
    """dequantize_tail (quantize.hpp:137-150): writes levels above stop_level
    of ``buffer`` in place."""
    _require_cuda(buffer, "buffer")
    return _dequantize(stream, plan, hierarchy, int(stop_level), buffer, ws)
