"""Fused-path diagnostics on the GPU box: per-level max error of decompose
against the CPU oracle, first bad index, for a list of shapes."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
import paper_2010_05872_b200 as mg  # noqa: E402
from oracle.oracle import Oracle  # noqa: E402

o = Oracle()
shapes = [(33, 33, 33), (65, 65, 65), (40, 36, 66), (35, 34, 100), (129, 65, 33), (17, 100, 64), (129, 129, 129)]
for dt in (np.float64, np.float32):
    for shape in shapes:
        rng = np.random.default_rng(1)
        x = rng.uniform(-10, 10, shape).astype(dt)
        h = mg.GridHierarchy.create(shape)
        L = h.num_levels()
        ws = mg.SolverWorkspace()
        got = mg.decompose(torch.from_numpy(x).cuda(), h, L - 1, ws).buffer.cpu().numpy().astype(np.float64)
        want = o.decompose(x, L - 1)
        nc = h.node_count(L - 1)
        e_coarse = np.abs(got[:nc] - want[:nc])
        e_shell = np.abs(got[nc:] - want[nc:])
        print(dt.__name__, shape, "shell max", e_shell.max(), "coarse max", e_coarse.max(), flush=True)
        if e_coarse.max() > 1e-6:
            bad = np.argwhere(e_coarse.reshape(h.level_dims(L - 1)) > 1e-6)
            print("   coarse bad count", len(bad), "first", bad[:5].tolist(), "last", bad[-3:].tolist())
        if e_shell.max() > 1e-6:
            bad = np.nonzero(e_shell > 1e-6)[0]
            print("   shell bad count", len(bad), "first", bad[:5].tolist())
        back = mg.recompose(mg.MultilevelCoefficients(torch.from_numpy(want.astype(dt)).cuda(), h, L - 1), ws).cpu().numpy()
        wr = o.recompose(want.astype(dt), shape, L - 1)
        er = np.abs(back.astype(np.float64) - wr)
        print("   rec max", er.max(), flush=True)
        if er.max() > 1e-6:
            bad = np.argwhere(er > 1e-6)
            print("   rec bad count", len(bad), "first", bad[:5].tolist())
