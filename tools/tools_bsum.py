"""Summarise a bench.py log: headline numbers and the top kernels (development helper)."""
import json
import sys

lines = [x for x in open(sys.argv[1]) if x.startswith("{")]
if not lines:
    print(open(sys.argv[1]).read()[-3000:])
    sys.exit(0)
d = json.loads(lines[-1])
print("ms_per_step", round(d["ms_per_step"], 4), "value", round(d["value"], 1), "step_frac",
      round(d.get("step_roofline", {}).get("frac", 0), 4))
print("roofline", {k: d["roofline"].get(k) for k in ("kernel", "kernel_ms", "frac")})
print("finest", d.get("finest_level_roofline"))
km = d.get("kernels_ms_per_step") or {}
print("profiled_step_ms", d.get("profiled_step_ms"), "sum", round(sum(km.values()), 4))
for k, v in sorted(km.items(), key=lambda x: -x[1])[:24]:
    print(f"  {k:28s} {v*1000:8.1f} us")
for k in ("batch", "quantize", "e2e", "clocks"):
    if k in d:
        print(k, {a: b for a, b in d[k].items() if not isinstance(b, str)})
