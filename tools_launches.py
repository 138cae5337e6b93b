"""Summarise gpurun_out/launches.csv (ncu --metrics gpu__time_duration.sum,dram__bytes_*)."""
import collections
import csv
import sys

path = sys.argv[1] if len(sys.argv) > 1 else "gpurun_out/launches.csv"
rows = list(csv.reader(open(path)))
hi = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
h = rows[hi]
ki, mi, vi, idi = h.index("Kernel Name"), h.index("Metric Name"), h.index("Metric Value"), h.index("ID")
per = collections.OrderedDict()
for r in rows[hi + 1:]:
    if len(r) <= vi:
        continue
    per.setdefault((int(r[idi]), r[ki]), {})[r[mi]] = float(r[vi].replace(",", ""))
items = list(per.items())
# last decompose+recompose step: from the last f3_dec_plane / k_dec_coef at the finest level
marks = [n for n, ((i, k), m) in enumerate(items) if "dec_plane" in k or "k_dec_coef" in k]
start = marks[-1]
while start > 0 and ("dec_plane" in items[start - 1][0][1] or "k_dec_coef" in items[start - 1][0][1] or
                     "col" in items[start - 1][0][1] or "sweep" in items[start - 1][0][1] or "apply" in items[start - 1][0][1]):
    start -= 1
tot = 0.0
agg = collections.OrderedDict()
for (i, k), m in items[start:]:
    name = k.split("(")[0].replace("void mgrx_b200::", "").replace("<unnamed>::", "")
    t = m.get("gpu__time_duration.sum", 0) / 1e3
    b = (m.get("dram__bytes_read.sum", 0) + m.get("dram__bytes_write.sum", 0)) / 1e6
    tot += t
    a = agg.setdefault(name, [0, 0.0, 0.0])
    a[0] += 1
    a[1] += t
    a[2] += b
    if "-v" in sys.argv:
        print(f"{i:5d} {name[:40]:40s} {t:9.1f} us {b:9.1f} MB {b / t * 1e-3 if t else 0:8.2f} TB/s")
print(f"step total {tot:.1f} us (serialised, cold)")
for name, (n, t, b) in sorted(agg.items(), key=lambda kv: -kv[1][1]):
    print(f"  {name[:40]:40s} x{n:3d} {t:9.1f} us {100 * t / tot:5.1f}%  {b:9.1f} MB")
