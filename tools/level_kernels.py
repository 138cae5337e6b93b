"""Per-kernel device times (library profiler, serialized launches) of one
decompose and one recompose of the bench field, grouped by level."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2010_05872_b200 as mg  # noqa: E402
from synthetic_fields import config2_field  # noqa: E402

arg = sys.argv[1] if len(sys.argv) > 1 else "513,513,513"
coords = None
if arg == "config3":
    from synthetic_fields import config3_field

    f, coords = config3_field(device="cuda")
elif arg == "config4b":
    from synthetic_fields import config4b_field

    f = config4b_field(device="cuda")
elif arg == "config4a":
    from synthetic_fields import config4a_field

    f = config4a_field(device="cuda")
else:
    f = config2_field(tuple(int(x) for x in arg.split(",")), seed=0, device="cuda")
h = mg.GridHierarchy.create(f.shape)
ws = mg.SolverWorkspace()
if coords is None:
    dec = lambda: mg.decompose(f, h, 0, ws)  # noqa: E731
    mc = dec()
    rec = lambda: mg.recompose(mc, ws)  # noqa: E731
else:
    dec = lambda: mg.decompose_nonuniform(f, h, coords, 0, ws)  # noqa: E731
    mc = dec()
    rec = lambda: mg.recompose_nonuniform(mc, coords, ws)  # noqa: E731
rec()
torch.cuda.synchronize()
for name, fn in (("decompose", dec), ("recompose", rec)):
    ws.profile_begin()
    for _ in range(5):
        fn()
    p = ws.profile_end()
    by = {}
    for k, (t, n) in p.items():
        lvl = int(k.split("@")[1]) if "@" in k else -1
        by.setdefault(lvl, []).append((k.split("@")[0], t / 5 * 1000, n // 5))
    print(name, "total %.1f us" % (sum(t for t, n in p.values()) / 5 * 1000))
    for lvl in sorted(by, reverse=True):
        tot = sum(x[1] for x in by[lvl])
        print(f"  level {lvl:2d} {tot:7.1f} us : " + "  ".join(f"{k} {t:.1f}" + (f"x{n}" if n > 1 else "") for k, t, n in by[lvl]))
