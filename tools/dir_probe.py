"""Decompose / recompose of the bench field timed three ways (eager, CUDA
graph, per-kernel profile) under the current environment: an A/B helper for
kernel-variant switches (MGRX_* env)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2010_05872_b200 as mg  # noqa: E402
from synthetic_fields import config2_field  # noqa: E402

dims = tuple(int(x) for x in (sys.argv[1] if len(sys.argv) > 1 else "513,513,513").split(","))
stop = int(sys.argv[2]) if len(sys.argv) > 2 else 0
f = config2_field(dims, seed=0, device="cuda")
h = mg.GridHierarchy.create(f.shape)
ws = mg.SolverWorkspace()
mc = mg.decompose(f, h, stop, ws)


def timed(fn, reps=20, graph=True):
    s = torch.cuda.Stream()
    with torch.cuda.stream(s):
        for _ in range(2):
            fn()
        torch.cuda.synchronize()
        g = None
        if graph:
            g = torch.cuda.CUDAGraph()
            with torch.cuda.graph(g, stream=s):
                fn()
            g.replay()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        ts = []
        for _ in range(reps):
            e0.record(s)
            g.replay() if graph else fn()
            e1.record(s)
            e1.synchronize()
            ts.append(e0.elapsed_time(e1))
    ts.sort()
    return ts[len(ts) // 2]


dec = lambda: mg.decompose(f, h, stop, ws)  # noqa: E731
rec = lambda: mg.recompose(mc, ws)  # noqa: E731
print(f"env {' '.join(k + '=' + v for k, v in os.environ.items() if k.startswith('MGRX'))}")
print(f"decompose graph {timed(dec):.4f} eager {timed(dec, graph=False):.4f} ms")
print(f"recompose graph {timed(rec):.4f} eager {timed(rec, graph=False):.4f} ms")
for name, fn in (("dec", dec), ("rec", rec)):
    ws.profile_begin()
    for _ in range(5):
        fn()
    p = ws.profile_end()
    items = sorted(p.items(), key=lambda kv: -kv[1][0])[:8]
    print(name, "  ".join(f"{k} {t / 5 * 1000:.1f}us" for k, (t, n) in items))
