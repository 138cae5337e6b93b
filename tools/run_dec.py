"""One warm-up and one measured decompose + recompose of a field (default
513^3 fp32) through the package: a short target for ncu."""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2010_05872_b200 as mg  # noqa: E402

shape = tuple(int(v) for v in (sys.argv[1] if len(sys.argv) > 1 else "513,513,513").split(","))
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 2
x = torch.randn(shape, device="cuda", dtype=torch.float32)
h = mg.GridHierarchy.create(shape)
ws = mg.SolverWorkspace()
for _ in range(reps):
    mc = mg.decompose(x, h, 0, ws)
    y = mg.recompose(mc, ws)
torch.cuda.synchronize()
print("ok", float((y - x).abs().max()))
