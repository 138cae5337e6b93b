"""Loader for the in-tree C-ABI library ``libmgrx_b200.so`` (include/mgrx_b200.h).

There is no fallback: if the library is missing the import fails loudly,
telling the caller to run ``__graft_entry__.build()``.
"""
from __future__ import annotations

import ctypes as C
import os

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("MGRX_LIB_PATH") or os.path.join(HERE, "libmgrx_b200.so")  # override: A/B builds (development)

# Every symbol include/mgrx_b200.h declares (checked by tests/test_abi.py).
EXPORTS = (
    "mgrx_abi_version", "mgrx_gpu_ctx_create", "mgrx_gpu_ctx_destroy", "mgrx_gpu_set_stream",
    "mgrx_gpu_get_stream", "mgrx_gpu_synchronize", "mgrx_gpu_last_error", "mgrx_gpu_launch_count",
    "mgrx_gpu_set_path", "mgrx_gpu_profile_begin", "mgrx_gpu_profile_end", "mgrx_hierarchy", "mgrx_make_plan", "mgrx_gpu_decompose", "mgrx_gpu_recompose",
    "mgrx_gpu_decompose_nonuniform", "mgrx_gpu_recompose_nonuniform", "mgrx_gpu_quantize",
    "mgrx_gpu_dequantize", "mgrx_gpu_decompose_quantize", "mgrx_gpu_dequantize_recompose", "mgrx_host_decompress", "mgrx_host_decompose", "mgrx_host_recompose", "mgrx_host_quantize", "mgrx_host_dequantize",
    "mgrx_gpu_workspace_size",
    "mgrx_gpu_choose_stop", "mgrx_host_decompose_adaptive", "mgrx_gpu_encode_labels", "mgrx_host_compress", "mgrx_gpu_field_stats", "mgrx_gpu_decompose_checked", "mgrx_host_lorenzo",
    "mgrx_gpu_slab_level", "mgrx_gpu_slab_dec_plane", "mgrx_gpu_slab_rec_plane", "mgrx_gpu_slab_inplane",
    "mgrx_gpu_slab_axis0", "mgrx_gpu_slab_apply", "mgrx_gpu_slab_interp", "mgrx_gpu_slab_pack", "mgrx_gpu_slab_unpack",
)

u64p = C.POINTER(C.c_uint64)
dp = C.POINTER(C.c_double)
vp = C.c_void_p


def _load() -> C.CDLL:
    if not os.path.exists(LIB_PATH):
        raise ImportError(
            f"{LIB_PATH} is missing: the CUDA extension has not been built "
            "(run `python -c 'import __graft_entry__ as g; g.build()'` or `make -C paper_2010_05872_b200/csrc`)")
    lib = C.CDLL(LIB_PATH)
    i = C.c_int
    sig = {
        "mgrx_abi_version": (i, []),
        "mgrx_gpu_ctx_create": (i, [i, C.POINTER(vp)]),
        "mgrx_gpu_ctx_destroy": (i, [vp]),
        "mgrx_gpu_set_stream": (i, [vp, vp]),
        "mgrx_gpu_get_stream": (vp, [vp]),
        "mgrx_gpu_synchronize": (i, [vp]),
        "mgrx_gpu_last_error": (C.c_char_p, [vp]),
        "mgrx_gpu_launch_count": (C.c_uint64, [vp]),
        "mgrx_gpu_set_path": (i, [vp, i]),
        "mgrx_gpu_profile_begin": (i, [vp]),
        "mgrx_gpu_profile_end": (i, [vp, C.c_char_p, dp, u64p, i, C.POINTER(i)]),
        "mgrx_hierarchy": (i, [i, u64p, i, C.POINTER(i), u64p, u64p]),
        "mgrx_make_plan": (i, [i, C.c_double, i, u64p, i, dp]),
        "mgrx_gpu_decompose": (i, [vp, i, i, u64p, i, i, vp, vp]),
        "mgrx_gpu_recompose": (i, [vp, i, i, u64p, i, i, vp, vp]),
        "mgrx_gpu_decompose_nonuniform": (i, [vp, i, i, u64p, i, i, C.POINTER(dp), vp, vp]),
        "mgrx_gpu_recompose_nonuniform": (i, [vp, i, i, u64p, i, i, C.POINTER(dp), vp, vp]),
        "mgrx_gpu_quantize": (i, [vp, i, i, u64p, i, i, dp, vp, vp, vp, vp, C.c_uint64, u64p]),
        "mgrx_gpu_dequantize": (i, [vp, i, i, u64p, i, i, dp, vp, vp, vp, C.c_uint64, vp]),
        "mgrx_gpu_decompose_quantize": (i, [vp, i, i, u64p, i, i, vp, dp, vp, vp, vp, vp, C.c_uint64, u64p]),
        "mgrx_gpu_dequantize_recompose": (i, [vp, i, i, u64p, i, i, dp, vp, vp, vp, C.c_uint64, vp, vp]),
        "mgrx_host_decompress": (i, [vp, i, i, u64p, i, i, dp, vp, vp, vp, C.c_uint64, vp, vp]),
        "mgrx_host_decompose": (i, [vp, i, i, u64p, i, i, vp, vp]),
        "mgrx_host_recompose": (i, [vp, i, i, u64p, i, i, vp, vp]),
        "mgrx_host_quantize": (i, [vp, i, i, u64p, i, i, dp, vp, vp, vp, vp, C.c_uint64, u64p]),
        "mgrx_host_dequantize": (i, [vp, i, i, u64p, i, i, dp, vp, vp, vp, C.c_uint64, vp]),
        "mgrx_gpu_workspace_size": (i, [i, i, u64p, i, i, u64p]),
        "mgrx_gpu_choose_stop": (i, [vp, i, i, u64p, vp, C.c_double, dp, C.c_double, i, dp, C.POINTER(i)]),
        "mgrx_host_decompose_adaptive": (i, [vp, i, i, u64p, i, vp, dp, dp, dp, i, i, vp, C.POINTER(i)]),
        "mgrx_gpu_encode_labels": (i, [vp, vp, C.c_uint64, vp, C.c_uint64, u64p]),
        "mgrx_host_compress": (i, [vp, i, i, u64p, i, vp, dp, i, i, dp, dp, dp, vp, C.c_uint64, u64p, u64p, vp,
                                   C.c_uint64, u64p, vp, C.POINTER(i)]),
        "mgrx_gpu_field_stats": (i, [vp, i, C.c_uint64, vp, dp, dp, u64p]),
        "mgrx_gpu_decompose_checked": (i, [vp, i, i, u64p, i, i, vp, vp, dp, dp, u64p]),
        "mgrx_host_lorenzo": (i, [vp, i, i, u64p, vp, C.c_double, vp, C.c_uint64, u64p, u64p, vp, C.c_uint64, u64p]),
        # slab mode (paper_2010_05872_b200/slab.py)
        "mgrx_gpu_slab_level": (i, [vp, i, i, u64p, i, i, C.POINTER(C.c_int64)]),
        "mgrx_gpu_slab_dec_plane": (i, [vp, i, i, u64p, i, i, C.c_uint64, C.c_uint64, vp, vp, vp, vp, C.c_int64]),
        "mgrx_gpu_slab_rec_plane": (i, [vp, i, i, u64p, i, i, C.c_uint64, C.c_uint64, vp, vp, C.c_int64]),
        "mgrx_gpu_slab_inplane": (i, [vp, i, i, u64p, i, i, C.c_uint64, C.c_uint64, vp]),
        "mgrx_gpu_slab_axis0": (i, [vp, i, i, u64p, i, i, C.c_uint64, vp]),
        "mgrx_gpu_slab_apply": (i, [vp, i, vp, vp, C.c_uint64, C.c_double]),
        "mgrx_gpu_slab_interp": (i, [vp, i, i, u64p, i, i, C.c_uint64, C.c_uint64, vp, vp, vp, C.c_int64]),
        "mgrx_gpu_slab_pack": (i, [vp, vp, C.c_uint64, C.c_uint64, u64p, i, vp]),
        "mgrx_gpu_slab_unpack": (i, [vp, vp, C.c_uint64, C.c_uint64, u64p, i, vp]),
    }
    for name, (res, args) in sig.items():
        f = getattr(lib, name)
        f.restype = res
        f.argtypes = args
    return lib


lib = _load()
