"""Diagnostics for the p2 passes: one level (stop = L - 1) of a small field,
shell and coarse blocks compared with the oracle, error locations."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2010_05872_b200 as mg  # noqa: E402
from oracle.oracle import Oracle  # noqa: E402

o = Oracle()
shape = tuple(int(v) for v in (sys.argv[1] if len(sys.argv) > 1 else "65,65,65").split(","))
kind = sys.argv[2] if len(sys.argv) > 2 else "rand"
rng = np.random.default_rng(1)
if kind == "rand":
    x = rng.uniform(-10, 10, shape).astype(np.float32)
elif kind == "ones":
    x = np.ones(shape, np.float32)
else:
    i, j, k = np.meshgrid(*[np.arange(n) for n in shape], indexing="ij")
    x = ((i % 2) * 1.0 + (j % 2) * 2.0 + (k % 2) * 4.0).astype(np.float32)
h = mg.GridHierarchy.create(shape)
L = h.num_levels()
stop = L - 1
ws = mg.SolverWorkspace()
want = o.decompose(x, stop)
got = mg.decompose(torch.from_numpy(x).cuda(), h, stop, ws).buffer.cpu().numpy().astype(np.float64)
nc = h.node_count(stop)
m = [(n + 1) // 2 for n in shape]
print("shape", shape, "L", L, "coarse", m, "range", float(x.max() - x.min()))
es = np.abs(got[nc:] - want[nc:])
print("shell max err", es.max(), "at", np.argmax(es), "count>1e-5", int((es > 1e-5).sum()), "of", es.size)
ec = np.abs(got[:nc] - want[:nc]).reshape(m)
print("coarse max err", ec.max(), "count>1e-5", int((ec > 1e-5).sum()), "of", ec.size)
if ec.max() > 1e-5:
    bad = np.argwhere(ec > 1e-5)
    print("coarse bad planes", np.unique(bad[:, 0])[:40])
    print("coarse bad rows", np.unique(bad[:, 1])[:40])
    print("coarse bad cols", np.unique(bad[:, 2])[:40])
    print("sample", [(tuple(b), got[:nc].reshape(m)[tuple(b)], want[:nc].reshape(m)[tuple(b)]) for b in bad[:5]])
    # the correction alone: got - x_nodal vs want - x_nodal
    xn = x[::2, ::2, ::2].astype(np.float64)
    zg = got[:nc].reshape(m) - xn
    zw = want[:nc].reshape(m) - xn
    print("z want absmax", np.abs(zw).max(), "z got absmax", np.abs(zg).max())
    for ax in range(3):
        sl = [slice(None)] * 3
        print("axis", ax, "err by index", np.round(np.abs(zg - zw).max(axis=tuple(a for a in range(3) if a != ax)), 4)[:20])
if es.max() > 1e-5:
    # locate shell errors: map shell offsets back through the oracle's layout
    bad = np.nonzero(es > 1e-5)[0][:10]
    print("shell bad offsets", bad, got[nc + bad], want[nc + bad])
if ec.max() > 1e-5:
    bad = ec > 1e-5
    print("bad per col", np.nonzero(bad.sum(axis=(0, 1)))[0].tolist()[:80])
    print("bad count per col", bad.sum(axis=(0, 1))[np.nonzero(bad.sum(axis=(0, 1)))[0]].tolist()[:80])
    print("bad count per row", bad.sum(axis=(0, 2)).tolist())
    print("bad count per plane", bad.sum(axis=(1, 2)).tolist())
