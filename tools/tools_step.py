"""One eager decompose + recompose step of the bench workload (513^3 fp32
config-2 field), after one warm-up step: the command profiled by
tools_prof.sh / tools_ncu_full.sh (no graph capture, no e2e pass)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2010_05872_b200 as mg  # noqa: E402
from synthetic_fields import config2_field  # noqa: E402

dims = tuple(int(x) for x in (sys.argv[1] if len(sys.argv) > 1 else "513,513,513").split(","))
f = config2_field(dims, seed=0, device="cuda")
h = mg.GridHierarchy.create(f.shape)
ws = mg.SolverWorkspace()
for _ in range(2):
    out = mg.recompose(mg.decompose(f, h, 0, ws), ws)
torch.cuda.synchronize()
# one level-wise quantize of the coefficients (tau = 1e-3 * range, budget tau / 4)
rg = float((f.max() - f.min()).item())
mg.quantize(mg.decompose(f, h, 0, ws), mg.make_plan(mg.QuantMode.levelwise, 1e-3 * rg / 4.0, h), ws)
torch.cuda.synchronize()
print("roundtrip linf", float((out - f).abs().max()))
