"""Marginal per-level cost of decompose / recompose in CUDA-graph replay
(development helper): for stop = L-1 .. 0, time a captured decompose and a
captured recompose of the bench field and print the increments."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2010_05872_b200 as mg  # noqa: E402
from synthetic_fields import config2_field  # noqa: E402

dims = tuple(int(x) for x in (sys.argv[1] if len(sys.argv) > 1 else "513,513,513").split(","))
f = config2_field(dims, seed=0, device="cuda")
h = mg.GridHierarchy.create(f.shape)
L = h.num_levels()


def timed(fn, reps=20):
    s = torch.cuda.Stream()
    with torch.cuda.stream(s):
        for _ in range(2):
            fn()
        torch.cuda.synchronize()
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g, stream=s):
            fn()
        g.replay()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        ts = []
        for _ in range(reps):
            e0.record(s)
            g.replay()
            e1.record(s)
            e1.synchronize()
            ts.append(e0.elapsed_time(e1))
    ts.sort()
    return ts[len(ts) // 2]


prev_d = prev_r = 0.0
print("stop  dec_ms  rec_ms  (marginal dec / rec of level stop+1)")
for stop in range(L - 1, -1, -1):
    ws = mg.SolverWorkspace()
    mc = mg.decompose(f, h, stop, ws)
    td = timed(lambda: mg.decompose(f, h, stop, ws))
    tr = timed(lambda: mg.recompose(mc, ws))
    print(f"{stop:4d} {td:7.4f} {tr:7.4f}   +{td - prev_d:.4f} +{tr - prev_r:.4f}")
    prev_d, prev_r = td, tr
