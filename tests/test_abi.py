"""CPU-side checks of the drop-in boundary: the C-ABI library loads, exports
every function include/mgrx_b200.h declares, and its host-only metadata
(GridHierarchy, make_plan) agrees with the oracle.  No device calls."""
import ctypes as C
import os
import re
import subprocess

import numpy as np
import pytest

import paper_2010_05872_b200 as mg
from paper_2010_05872_b200._lib import EXPORTS, LIB_PATH, lib
from oracle.oracle import Oracle

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "mgrx_b200.h")


def declared_functions():
    src = open(HEADER).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(mgrx_[a-z0-9_]+)\s*\(", src)))


def test_header_declares_what_the_binding_lists():
    assert declared_functions() == sorted(EXPORTS)


def test_library_exports_every_declared_symbol():
    out = subprocess.run(["nm", "-D", "--defined-only", LIB_PATH], capture_output=True, text=True, check=True).stdout
    exported = set(re.findall(r" T (mgrx_[a-z0-9_]+)", out))
    missing = [f for f in declared_functions() if f not in exported]
    assert not missing, missing
    for f in declared_functions():
        assert hasattr(lib, f)


def test_library_is_sm100a_only():
    out = subprocess.run(["/usr/local/cuda/bin/cuobjdump", "--list-elf", LIB_PATH], capture_output=True, text=True)
    archs = set(re.findall(r"sm_(\d+a?)", out.stdout))
    assert archs == {"100a"}, archs


def test_abi_version():
    assert lib.mgrx_abi_version() == 1


@pytest.mark.parametrize("dims,levels", [((65, 65, 65), 4), ((100, 500, 500), None), ((5,), None), ((513,) * 3, None),
                                         ((288, 115, 69, 69), None), ((4097, 4097), None), ((2, 2), None),
                                         ((3, 1025), None), ((1025,) * 3, None)])
def test_hierarchy_matches_oracle(dims, levels):
    o = Oracle()
    L, ld, dc = o.hierarchy(dims, levels)
    h = mg.GridHierarchy.create(dims, levels)
    assert h.num_levels() == L
    assert [h.level_dims(l) for l in range(L + 1)] == ld
    assert h.delta_counts() == dc
    assert h.total_count() == int(np.prod(dims))
    for mode in (0, 1):
        p = mg.make_plan(mg.QuantMode(mode), 1e-3, h)
        assert p.bin_widths.tobytes() == o.make_plan(mode, 1e-3, dims, levels).tobytes()


def test_error_codes_mirror_errc():
    with pytest.raises(mg.Error) as e:
        mg.GridHierarchy.create((1, 5))
    assert e.value.code == "invalid_dims"
    with pytest.raises(mg.Error) as e:
        mg.GridHierarchy.create((5, 5), 3)
    assert e.value.code == "depth_exceeded"
    with pytest.raises(mg.Error) as e:
        mg.GridHierarchy.create(())
    assert e.value.code == "invalid_dims"
    h = mg.GridHierarchy.create((5, 5))
    with pytest.raises(mg.Error) as e:
        h.delta_count(3)
    assert e.value.code == "invalid_level"
    for bad in (0.0, -1.0, float("nan"), float("inf")):
        with pytest.raises(mg.Error) as e:
            mg.make_plan(mg.QuantMode.uniform, bad, h)
        assert e.value.code == "invalid_budget"
    # rank above MGRX_MAX_DIMS
    with pytest.raises(mg.Error):
        mg.GridHierarchy.create((3,) * 9)


def test_null_context_is_rejected():
    dims = (C.c_uint64 * 1)(5)
    assert lib.mgrx_gpu_decompose(None, 0, 1, dims, -1, 0, None, None) == 102
    assert lib.mgrx_gpu_last_error(None) == b"null context"
