"""Quantize / dequantize of the bench field's coefficients: per-kernel
device times (library profiler) and whole-call CUDA-event times."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2010_05872_b200 as mg  # noqa: E402
from synthetic_fields import config2_field  # noqa: E402

f = config2_field(seed=0, device="cuda")
h = mg.GridHierarchy.create(f.shape)
ws = mg.SolverWorkspace()
mc = mg.decompose(f, h, 0, ws)
rg = float((f.max() - f.min()).item())
for t in (1e-2, 1e-3, 1e-4):
    plan = mg.make_plan(mg.QuantMode.levelwise, t * rg / 4.0, h)
    for _ in range(2):
        s = mg.quantize(mc, plan, ws)
        d = mg.dequantize(s, plan, h, ws)
    torch.cuda.synchronize()
    e = [torch.cuda.Event(enable_timing=True) for _ in range(3)]
    e[0].record()
    for _ in range(10):
        s = mg.quantize(mc, plan, ws)
    e[1].record()
    for _ in range(10):
        d = mg.dequantize(s, plan, h, ws)
    e[2].record()
    torch.cuda.synchronize()
    ws.profile_begin()
    s = mg.quantize(mc, plan, ws)
    d = mg.dequantize(s, plan, h, ws)
    p = ws.profile_end()
    print(f"tau {t:g}: quantize {e[0].elapsed_time(e[1]) / 10:.4f} ms, dequantize {e[1].elapsed_time(e[2]) / 10:.4f} ms,"
          f" outliers {s.outlier_positions.numel()};", "  ".join(f"{k} {v[0] * 1000:.1f}us" for k, v in p.items()))
