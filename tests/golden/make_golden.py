"""Generates tests/golden/golden.npz from the UNMODIFIED reference.

Run in the build container (needs /root/reference, compiled by
`make -C oracle ref`):  python tests/golden/make_golden.py

The reference ships no fixture files; its tests generate inputs
in-test.  The fixtures here are (a) the reference tests' stated known
answers, recomputed through the reference library, and (b) reference outputs
(decompose / recompose / quantize / dequantize / one level step) on seeded
inputs over the shapes the reference's own tests use
(test_transform.cpp:303,358-363,399; test_reorder.cpp:299).  The oracle and
the GPU path are checked against these bytes.
"""
from __future__ import annotations

import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, ROOT)

from oracle.oracle import Reference  # noqa: E402

SHAPES = [
    (17, 17, 17), (9, 33, 17), (5, 5, 5, 5), (33, 33), (65,), (12, 20), (6, 6, 6), (31, 14, 9), (2, 2),
    (100, 11), (17, 9, 5), (6, 9, 4), (9, 7), (17,), (9, 9), (33, 5), (9, 9, 9), (33, 17), (3, 1025),
    (8,), (6, 4), (5, 5, 5), (2, 3, 4, 5, 3), (24, 10, 12),
]


def key(shape, *parts):
    return "x".join(str(s) for s in shape) + "_" + "_".join(str(p) for p in parts)


def main():
    ref = Reference()
    rng = np.random.default_rng(20240601)
    out = {}
    for shape in SHAPES:
        L = ref.hierarchy(shape)[0]
        for dt in (np.float64, np.float32):
            name = "f64" if dt == np.float64 else "f32"
            x = rng.uniform(-100, 100, shape).astype(dt)
            out[key(shape, name, "in")] = x
            for stop in sorted({0, min(1, L), L}):
                c = ref.decompose(x, stop)
                out[key(shape, name, "dec", stop)] = c
                out[key(shape, name, "rec", stop)] = ref.recompose(c, shape, stop)
            # quantization at a budget that yields outliers on coarse levels
            q = ref.make_plan(1, 1e-3 * 200.0, shape)
            c0 = out[key(shape, name, "dec", 0)]
            lab, opos, oval = ref.quantize(c0, shape, q)
            out[key(shape, name, "q")] = q
            out[key(shape, name, "labels")] = lab
            out[key(shape, name, "opos")] = opos
            out[key(shape, name, "oval")] = oval
            out[key(shape, name, "deq")] = ref.dequantize(lab, opos, oval, shape, q, dtype=dt)
            if L >= 2:
                lab, opos, oval = ref.quantize(c0, shape, q, stop=1)
                out[key(shape, name, "qtail_labels")] = lab
                out[key(shape, name, "qtail_opos")] = opos
    # one level step (reorder + coefficients + correction) at the finest level
    for shape in [(9, 9), (17, 9, 5), (6, 5, 3), (7, 4), (9,)]:
        x = rng.uniform(-2, 2, shape)
        L = ref.hierarchy(shape)[0]
        f, corr = ref.level_step(x, L)
        out[key(shape, "step_in")] = x
        out[key(shape, "step_field")] = f
        out[key(shape, "step_corr")] = corr
    # strided-reference decomposition (reference.hpp:237) — bitwise equal
    for shape in [(17, 17), (9, 9, 9), (33, 5), (6, 9, 4)]:
        x = rng.uniform(-8, 8, shape)
        out[key(shape, "strided_in")] = x
        out[key(shape, "strided_dec")] = ref.strided_decompose(x)

    # ---- stated known answers of the reference tests ----------------------
    out["ka_load_zero"] = ref.load_vector_1d([0, 0, 0, 0, 0])                  # test_transform.cpp:37
    out["ka_load_ones"] = ref.load_vector_1d([1, 1, 1, 1, 1])                  # :40 -> (1,2,1)
    out["ka_load_pure1d"] = ref.load_vector_1d([0, 1, 0, 1, 0])                # :46 -> (.5,1,.5)
    out["ka_solve_ones_rhs"] = ref.solve_correction_1d(
        [(2 / 3 if i in (0, 6) else 4 / 3) + (1 / 3 if i > 0 else 0) + (1 / 3 if i < 6 else 0) for i in range(7)])
    out["ka_solve_2x2"] = ref.solve_correction_1d([1.0, 1.0])                  # :118
    out["ka_reorder_5"] = ref.reorder_pack(np.arange(10.0, 15.0), stop=1)      # test_reorder.cpp:193 path
    out["ka_grid_65_4"] = np.array(ref.hierarchy((65, 65, 65), 4)[2], dtype=np.uint64)  # test_grid.cpp:330
    out["ka_levels_100x500x500"] = np.array([ref.hierarchy((100, 500, 500))[0]])       # :340 -> 6
    out["ka_delta_5"] = np.array(ref.hierarchy((5,))[2], dtype=np.uint64)             # :347 -> 2,1,2
    out["ka_plan_lw_65_4"] = ref.make_plan(1, 0.125, (65, 65, 65), 4)                  # test_quantize.cpp:31
    out["ka_plan_uni_65_4"] = ref.make_plan(0, 0.125, (65, 65, 65), 4)                 # :28
    for k in list(out):
        if out[k].dtype == np.uint64 and not k.startswith("ka_"):
            out[k] = out[k].astype(np.int64)
    np.savez_compressed(os.path.join(HERE, "golden.npz"), **out)
    print(f"wrote {len(out)} arrays to {os.path.join(HERE, 'golden.npz')}")


if __name__ == "__main__":
    main()
