"""Small invocation of every kernel family (fused 3-D passes incl. the 3-CTA
variants, row / column passes, tail, general per-step path, nonuniform path,
quantize / dequantize, adaptive stop, label coding, Lorenzo, field stats)
for compute-sanitizer runs (tools/sanitize.sh).  Shapes are small so the
tools finish in minutes; the fused levels are forced with
MGRX_FUSED_MIN_ELEMS=1 (set by the script)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2010_05872_b200 as mg  # noqa: E402
from synthetic_fields import nonuniform_coords  # noqa: E402

rng = np.random.default_rng(0)
shapes = [((65, 65, 65), np.float32), ((33, 40, 70), np.float64), ((17, 12, 1079), np.float32),
          ((129, 65, 33), np.float32), ((17, 12), np.float64), ((9, 8, 7, 6), np.float32)]
ws = mg.SolverWorkspace()
for shape, dt in shapes:
    x = torch.from_numpy(rng.uniform(-1, 1, shape).astype(dt)).cuda()
    h = mg.GridHierarchy.create(shape)
    mc = mg.decompose(x, h, 0, ws)
    y = mg.recompose(mc, ws)
    plan = mg.make_plan(mg.QuantMode.levelwise, 1e-3, h)
    s = mg.quantize(mc, plan, ws)
    mg.recompose(mg.dequantize(s, plan, h, ws), ws)
    if h.num_levels() >= 2:
        mg.recompose(mg.decompose(x, h, 1, ws), ws)
    torch.cuda.synchronize()
    print("ok", shape, float((y - x).abs().max()), flush=True)
# nonuniform path
shape = (33, 20)
coords = [nonuniform_coords(n, seed=1, axis=a) for a, n in enumerate(shape)]
x = torch.from_numpy(rng.uniform(-1, 1, shape)).cuda()
h = mg.GridHierarchy.create(shape)
mc = mg.decompose_nonuniform(x, h, coords, 0, ws)
mg.recompose_nonuniform(mc, coords, ws)
torch.cuda.synchronize()
print("ok nonuniform", flush=True)
