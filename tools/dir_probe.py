"""Decompose / recompose of the bench field timed three ways (eager, CUDA
graph, per-kernel profile) under the current environment: an A/B helper for
kernel-variant switches (MGRX_* env)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2010_05872_b200 as mg  # noqa: E402
from synthetic_fields import config2_field  # noqa: E402

arg = sys.argv[1] if len(sys.argv) > 1 else "513,513,513"
stop = int(sys.argv[2]) if len(sys.argv) > 2 else 0
coords = None
if arg.startswith("config"):
    import synthetic_fields as sf

    f = getattr(sf, arg + "_field")(device="cuda")
    if isinstance(f, tuple):
        f, coords = f
else:
    f = config2_field(tuple(int(x) for x in arg.split(",")), seed=0, device="cuda")
h = mg.GridHierarchy.create(f.shape)
ws = mg.SolverWorkspace()
if coords is None:
    mc = mg.decompose(f, h, stop, ws)
else:
    mc = mg.decompose_nonuniform(f, h, coords, stop, ws)


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


if coords is None:
    dec = lambda: mg.decompose(f, h, stop, ws)  # noqa: E731
    rec = lambda: mg.recompose(mc, ws)  # noqa: E731
else:
    dec = lambda: mg.decompose_nonuniform(f, h, coords, stop, ws)  # noqa: E731
    rec = lambda: mg.recompose_nonuniform(mc, coords, ws)  # noqa: E731
nbytes = sum(2 * f.element_size() * h.node_count(l) for l in range(stop + 1, h.num_levels() + 1))
print(f"env {' '.join(k + '=' + v for k, v in os.environ.items() if k.startswith('MGRX'))}")
td, tr = timed(dec), timed(rec)
print(f"decompose graph {td:.4f} eager {timed(dec, graph=False):.4f} ms  ({nbytes / td / 1e6:.0f} GB/s alg, "
      f"{nbytes / td / 1e6 / 6551.7:.3f} of peak)")
print(f"recompose graph {tr:.4f} eager {timed(rec, graph=False):.4f} ms  ({nbytes / tr / 1e6:.0f} GB/s alg, "
      f"{nbytes / tr / 1e6 / 6551.7:.3f} of peak)")
for name, fn in (("dec", dec), ("rec", rec)):
    ws.profile_begin()
    for _ in range(5):
        fn()
    p = ws.profile_end()
    items = sorted(p.items(), key=lambda kv: -kv[1][0])[:8]
    print(name, "  ".join(f"{k} {t / 5 * 1000:.1f}us" for k, (t, n) in items))
