"""TEST INFRASTRUCTURE ONLY — ctypes bindings to the CPU checkers.

* ``Oracle``    -> oracle/libmgrx_oracle.so, our plain-C restatement
                   (oracle/mgrx_oracle.c) of the reference hot path.
* ``Reference`` -> oracle/_ref/libmgrx_ref.so, the unmodified reference
                   (/root/reference/proj/core) compiled by oracle/Makefile.

Only tests/, ``__graft_entry__.smoke()`` and bench.py's CPU-baseline leg may
import this module.  Both libraries expose the same call shapes, so the tests
can swap one for the other.  Non-zero status codes are 1 + mgrx::errc
(error.hpp:9-36) and are raised as :class:`OracleError`.
"""
from __future__ import annotations

import ctypes as C
import os

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ORACLE_SO = os.path.join(HERE, "libmgrx_oracle.so")
REF_SO = os.path.join(HERE, "_ref", "libmgrx_ref.so")

ERRC = [
    "invalid_dims", "depth_exceeded", "invalid_level", "invalid_axis", "degenerate_line",
    "degenerate_system", "shape_error", "invalid_budget", "nonfinite_data", "decode_error",
    "not_an_artifact", "unsupported_version", "corrupt", "undefined_psnr", "invalid_input",
]


class OracleError(RuntimeError):
    def __init__(self, status: int, msg: str = ""):
        self.status = status
        self.errc = ERRC[status - 1] if 1 <= status <= len(ERRC) else f"status{status}"
        super().__init__(f"{self.errc}: {msg}")


_u64p = C.POINTER(C.c_uint64)
_dp = C.POINTER(C.c_double)
_fp = C.POINTER(C.c_float)
_ip = C.POINTER(C.c_int32)


def _ptr(a: np.ndarray):
    return a.ctypes.data_as(C.c_void_p)


def _dims(dims):
    a = np.ascontiguousarray(np.asarray(dims, dtype=np.uint64))
    return a, a.ctypes.data_as(_u64p)


class _Lib:
    prefix = ""
    path = ""

    def __init__(self):
        if not os.path.exists(self.path):
            raise FileNotFoundError(f"{self.path} not built (run `make -C oracle oracle ref`)")
        self.lib = C.CDLL(self.path)

    def _fn(self, name):
        f = getattr(self.lib, self.prefix + name)
        f.restype = C.c_int
        return f

    def _check(self, rc):
        if rc != 0:
            msg = ""
            if hasattr(self.lib, "ref_last_error"):
                self.lib.ref_last_error.restype = C.c_char_p
                msg = (self.lib.ref_last_error() or b"").decode()
            raise OracleError(rc, msg)

    # -- grid ---------------------------------------------------------------
    def hierarchy(self, dims, levels=None):
        """(L, level_dims[L+1][d] coarsest first, delta_counts[L+1])."""
        d, dp = _dims(dims)
        L = C.c_int()
        ld = np.zeros((70, len(d)), dtype=np.uint64)
        dc = np.zeros(70, dtype=np.uint64)
        self._check(self._fn("hierarchy")(len(d), dp, -1 if levels is None else levels, C.byref(L),
                                          ld.ctypes.data_as(_u64p), dc.ctypes.data_as(_u64p)))
        n = L.value + 1
        return L.value, [tuple(int(x) for x in r) for r in ld[:n]], [int(x) for x in dc[:n]]

    def make_plan(self, mode, budget, dims, levels=None):
        d, dp = _dims(dims)
        q = np.zeros(70, dtype=np.float64)
        self._check(self._fn("make_plan")(C.c_int(mode), C.c_double(budget), len(d), dp,
                                          -1 if levels is None else levels, q.ctypes.data_as(_dp)))
        L = self.hierarchy(dims, levels)[0]
        return q[: L + 1].copy()

    # -- 1-D kernels --------------------------------------------------------
    def load_vector_1d(self, line):
        line = np.ascontiguousarray(line, dtype=np.float64)
        out = np.zeros((len(line) + 1) // 2)
        self._check(self._fn("load_vector_1d")(line.ctypes.data_as(_dp), C.c_uint64(len(line)),
                                               out.ctypes.data_as(_dp)))
        return out

    def solve_correction_1d(self, f):
        f = np.array(f, dtype=np.float64)
        self._check(self._fn("solve_correction_1d")(f.ctypes.data_as(_dp), C.c_uint64(len(f))))
        return f

    def thomas_aux(self, m):
        w = np.zeros(m)
        inv = np.zeros(m)
        self._check(self._fn("thomas_aux")(C.c_uint64(m), w.ctypes.data_as(_dp), inv.ctypes.data_as(_dp)))
        return w, inv

    # -- transform ----------------------------------------------------------
    def _sfx(self, a):
        return "f32" if a.dtype == np.float32 else "f64"

    def decompose(self, field, stop=0, levels=None, batch=32):
        field = np.ascontiguousarray(field)
        d, dp = _dims(field.shape)
        out = np.empty(field.size, dtype=field.dtype)
        args = [len(d), dp, -1 if levels is None else levels, stop, _ptr(field), _ptr(out)]
        if self.prefix == "ref_":
            args.append(batch)
        self._check(self._fn("decompose_" + self._sfx(field))(*args))
        return out

    def recompose(self, buf, dims, stop=0, levels=None):
        buf = np.ascontiguousarray(buf)
        d, dp = _dims(dims)
        out = np.empty(int(np.prod(dims)), dtype=buf.dtype)
        self._check(self._fn("recompose_" + self._sfx(buf))(len(d), dp, -1 if levels is None else levels,
                                                           stop, _ptr(buf), _ptr(out)))
        return out.reshape(tuple(dims))

    def quantize(self, buf, dims, q, stop=0, levels=None):
        """(labels concatenated per level, outlier positions, outlier values)."""
        buf = np.ascontiguousarray(buf)
        d, dp = _dims(dims)
        q = np.ascontiguousarray(q, dtype=np.float64)
        L, _, dc = self.hierarchy(dims, levels)
        nlab = sum(dc[stop + 1:]) if stop > 0 else sum(dc)
        labels = np.zeros(nlab, dtype=np.int32)
        cap = buf.size
        opos = np.zeros(cap, dtype=np.uint64)
        oval = np.zeros(cap, dtype=buf.dtype)
        n = C.c_uint64()
        self._check(self._fn("quantize_" + self._sfx(buf))(
            len(d), dp, -1 if levels is None else levels, stop, q.ctypes.data_as(_dp), _ptr(buf),
            labels.ctypes.data_as(_ip), opos.ctypes.data_as(_u64p), _ptr(oval), C.c_uint64(cap), C.byref(n)))
        return labels, opos[: n.value].copy(), oval[: n.value].copy()

    def dequantize(self, labels, opos, oval, dims, q, stop=0, levels=None, dtype=np.float64, base=None):
        d, dp = _dims(dims)
        q = np.ascontiguousarray(q, dtype=np.float64)
        labels = np.ascontiguousarray(labels, dtype=np.int32)
        opos = np.ascontiguousarray(opos, dtype=np.uint64)
        oval = np.ascontiguousarray(oval, dtype=dtype)
        out = np.zeros(int(np.prod(dims)), dtype=dtype) if base is None else np.array(base, dtype=dtype)
        self._check(self._fn("dequantize_" + ("f32" if np.dtype(dtype) == np.float32 else "f64"))(
            len(d), dp, -1 if levels is None else levels, stop, q.ctypes.data_as(_dp),
            labels.ctypes.data_as(_ip), opos.ctypes.data_as(_u64p), _ptr(oval), C.c_uint64(len(opos)),
            _ptr(out)))
        return out


class Oracle(_Lib):
    prefix = "mo_"
    path = ORACLE_SO

    def _coords(self, coords):
        arrs = [np.ascontiguousarray(c, dtype=np.float64) for c in coords]
        ptrs = (_dp * len(arrs))(*[a.ctypes.data_as(_dp) for a in arrs])
        return arrs, ptrs

    def decompose_nu(self, field, coords, stop=0, levels=None):
        field = np.ascontiguousarray(field)
        d, dp = _dims(field.shape)
        keep, ptrs = self._coords(coords)
        out = np.empty(field.size, dtype=field.dtype)
        self._check(self._fn("decompose_nu_" + self._sfx(field))(
            len(d), dp, -1 if levels is None else levels, stop, ptrs, _ptr(field), _ptr(out)))
        return out

    def recompose_nu(self, buf, dims, coords, stop=0, levels=None):
        buf = np.ascontiguousarray(buf)
        d, dp = _dims(dims)
        keep, ptrs = self._coords(coords)
        out = np.empty(int(np.prod(dims)), dtype=buf.dtype)
        self._check(self._fn("recompose_nu_" + self._sfx(buf))(
            len(d), dp, -1 if levels is None else levels, stop, ptrs, _ptr(buf), _ptr(out)))
        return out.reshape(tuple(dims))

    def load_vector_nu_1d(self, line, x):
        line = np.ascontiguousarray(line, dtype=np.float64)
        x = np.ascontiguousarray(x, dtype=np.float64)
        out = np.zeros((len(line) + 1) // 2)
        self._check(self._fn("load_vector_nu_1d")(line.ctypes.data_as(_dp), x.ctypes.data_as(_dp),
                                                  C.c_uint64(len(line)), out.ctypes.data_as(_dp)))
        return out

    def solve_correction_nu_1d(self, f, X):
        f = np.array(f, dtype=np.float64)
        X = np.ascontiguousarray(X, dtype=np.float64)
        self._check(self._fn("solve_correction_nu_1d")(f.ctypes.data_as(_dp), X.ctypes.data_as(_dp),
                                                       C.c_uint64(len(f))))
        return f


class Reference(_Lib):
    prefix = "ref_"
    path = REF_SO

    def strided_decompose(self, field, stop=0, levels=None):
        field = np.ascontiguousarray(field, dtype=np.float64)
        d, dp = _dims(field.shape)
        out = np.empty(field.size)
        self._check(self._fn("strided_decompose_f64")(len(d), dp, -1 if levels is None else levels, stop,
                                                      _ptr(field), _ptr(out)))
        return out

    def level_step(self, field, level):
        """reorder_level + compute_coefficients + compute_correction at `level`
        on a natural-order field; returns (reordered field, correction)."""
        field = np.array(field)
        d, dp = _dims(field.shape)
        _, ld, _ = self.hierarchy(field.shape)
        corr = np.zeros(int(np.prod(ld[level - 1])))
        fn = self._fn("level_step_" + self._sfx(field))
        self._check(fn(len(d), dp, level, _ptr(field), corr.ctypes.data_as(_dp)))
        return field, corr.reshape(ld[level - 1])

    def lorenzo(self, block, e):
        """compress_lorenzo (lorenzo.hpp:87-128) -> (labels, outlier positions, outlier values)."""
        block = np.ascontiguousarray(block)
        d, dp = _dims(block.shape)
        labels = np.empty(block.size, np.int32)
        cap = block.size
        opos = np.empty(cap, np.uint64)
        oval = np.empty(cap, block.dtype)
        n = C.c_uint64(0)
        fn = self._fn("lorenzo_" + self._sfx(block))
        self._check(fn(len(d), dp, _ptr(block), C.c_double(e), labels.ctypes.data_as(C.c_void_p),
                       opos.ctypes.data_as(C.c_void_p), _ptr(oval), C.c_uint64(cap), C.byref(n)))
        return labels, opos[:n.value], oval[:n.value]

    def encode_labels(self, labels):
        """encode_labels (src/huffman.cpp:209-255) -> bytes."""
        labels = np.ascontiguousarray(labels, dtype=np.int32)
        cap = 32 + 4 * labels.size + (1 << 17) + 64
        out = np.empty(cap, dtype=np.uint8)
        size = C.c_uint64(0)
        self._check(self._fn("encode_labels")(labels.ctypes.data_as(C.c_void_p), C.c_uint64(labels.size),
                                              out.ctypes.data_as(C.c_void_p), C.c_uint64(cap), C.byref(size)))
        return out[:size.value].tobytes()

    def choose_stop(self, block, e, interp_penalty, lorenzo_penalty, step=8):
        """The reference's accumulate_block_errors + choose_stop decision
        (adaptive.hpp:51-104) on a natural-order level block: returns
        (stop, lorenzo_total, interp_total)."""
        block = np.ascontiguousarray(block)
        d, dp = _dims(block.shape)
        pen = np.ascontiguousarray(np.asarray(interp_penalty, dtype=np.float64))
        tot = np.zeros(2)
        stop = C.c_int(0)
        fn = self._fn("choose_stop_" + self._sfx(block))
        self._check(fn(len(d), dp, _ptr(block), C.c_double(e), pen.ctypes.data_as(_dp), C.c_double(lorenzo_penalty),
                       int(step), tot.ctypes.data_as(_dp), C.byref(stop)))
        return bool(stop.value), float(tot[0]), float(tot[1])

    def reorder_pack(self, field, stop=0):
        field = np.ascontiguousarray(field, dtype=np.float64)
        d, dp = _dims(field.shape)
        out = np.empty(field.size)
        self._check(self._fn("reorder_pack_f64")(len(d), dp, stop, _ptr(field), _ptr(out)))
        return out

    def estimated_cost(self, mode, budget, dims, range_, levels=None):
        d, dp = _dims(dims)
        out = C.c_double()
        self._check(self._fn("estimated_cost")(C.c_int(mode), C.c_double(budget), len(d), dp,
                                               -1 if levels is None else levels, C.c_double(range_),
                                               C.byref(out)))
        return out.value


def reference_available() -> bool:
    return os.path.exists(REF_SO)
