"""Parity bars shared by the tests and bench.py's cpu_baseline leg (TEST
INFRASTRUCTURE: the checker, never the product path).

north_star's label bar: quantized indices bit-exact, except values within
1 ulp of a bin edge; count and report those.  A label produced from the
GPU's coefficient may differ from the reference's only where the
reference's coefficient v lies within `ulps` ulp_T(v) of an edge
(k + 1/2) q_l of the rounding r = nearbyint(double(v) / q_l)
(quantize_span, reference proj/core/include/mgrx/quantize.hpp:58-73).
"""
from __future__ import annotations

import numpy as np


def label_flips(want, got_labels, ref_labels, delta_counts, q, ulps=1.0):
    """(count, worst distance in ulp) of label differences; raises
    AssertionError when one is farther than `ulps` ulp from its bin edge.

    want          the reference's coefficients (level-centric, dtype T)
    got_labels    labels quantized from the GPU's coefficients
    ref_labels    the reference's labels of `want`
    delta_counts  #N*_l, l = 0..L (labels are concatenated coarsest first)
    q             bin widths q_l, l = 0..L
    """
    got_labels = np.asarray(got_labels)
    ref_labels = np.asarray(ref_labels)
    diff = np.nonzero(got_labels != ref_labels)[0]
    if diff.size == 0:
        return 0, 0.0
    v = np.asarray(want)[diff]
    lvl = np.searchsorted(np.cumsum(delta_counts), diff, side="right")
    ql = np.asarray(q, dtype=np.float64)[lvl]
    r = np.abs(v.astype(np.float64) / ql)
    dist = np.abs(r - np.floor(r) - 0.5) * ql  # distance of |v| from the nearest edge (k + 1/2) q
    ulp = np.spacing(np.abs(v)).astype(np.float64)
    in_ulps = dist / np.maximum(ulp, 1e-300)
    worst = float(in_ulps.max())
    bad = in_ulps > ulps
    assert not bad.any(), (
        f"{int(bad.sum())} of {diff.size} label differences lie farther than {ulps} ulp from a bin edge "
        f"(worst {worst:.3g} ulp; positions {diff[bad][:8].tolist()})")
    return int(diff.size), worst
