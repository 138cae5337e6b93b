"""Summarise gpurun_out/launches.csv (ncu --metrics gpu__time_duration.sum,dram__bytes_*) per kernel."""
import collections
import sys

from tools_ncu_csv import last_step, nbytes, read_launches, short

path = sys.argv[1] if len(sys.argv) > 1 else "gpurun_out/launches.csv"
step = last_step(read_launches(path))
agg = collections.OrderedDict()
for i, k, m in step:
    a = agg.setdefault(short(k), [0, 0.0, 0.0])
    a[0] += 1
    a[1] += m.get("gpu__time_duration.sum", 0) * 1e6
    a[2] += nbytes(m) / 1e6
tot = sum(a[1] for a in agg.values())
print(f"step total {tot:.1f} us (serialised, cold)")
for name, (n, t, b) in sorted(agg.items(), key=lambda kv: -kv[1][1]):
    print(f"  {name:40s} x{n:3d} {t:9.1f} us {100 * t / tot:5.1f}% {b:11.1f} MB")
