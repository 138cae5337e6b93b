"""Turn an ncu launch list (gpu__time_duration + dram bytes) into the
committed per-round summary: profiles/<round>_launches.md and
profiles/traffic.json (DRAM bytes per launch of each kernel@level, used by
bench.py for roofline.traffic).  Kernel@level is recovered from launch order
of one decompose+recompose step (the last one in the list)."""
import collections
import csv
import json
import sys

src, rnd = sys.argv[1], sys.argv[2]
rows = list(csv.reader(open(src)))
hi = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
h = rows[hi]
ki, mi, vi, idi = h.index("Kernel Name"), h.index("Metric Name"), h.index("Metric Value"), h.index("ID")
per = collections.OrderedDict()
for r in rows[hi + 1:]:
    if len(r) <= vi:
        continue
    per.setdefault((int(r[idi]), r[ki]), {})[r[mi]] = float(r[vi].replace(",", ""))
items = list(per.items())
# last step: from the last launch of the finest-level decompose plane kernel
starts = [n for n, ((i, k), m) in enumerate(items) if "k_f3_dec_plane" in k]
# the finest-level plane kernel is the first of a run of dec planes
first_of_run = [n for n in starts if n == 0 or "k_f3_dec_plane" not in items[n - 3][0][1]]
start = first_of_run[-1]
step = items[start:]
# decompose levels L..., recompose ...; tag by order of appearance per kernel name
L = 9
names = []
dec_level = {}
counter = collections.Counter()
out_rows = []
traffic = {}
for (i, k), m in step:
    name = k.split("(")[0].replace("void mgrx_b200::", "").replace("<unnamed>::", "")
    base = name.split("<")[0]
    t = m.get("gpu__time_duration.sum", 0) / 1e3
    rd = m.get("dram__bytes_read.sum", 0)
    wr = m.get("dram__bytes_write.sum", 0)
    out_rows.append((i, name, t, rd, wr))
tot = sum(r[2] for r in out_rows)
with open(f"profiles/{rnd}_launches.md", "w") as f:
    f.write(f"# {rnd}: ncu launch list, one decompose + recompose step of the 513^3 fp32 bench\n\n")
    f.write("Command: `ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum "
            "--clock-control none python bench.py --steps 2 --warmup 1 --no-cpu-baseline` (tools_prof.sh).\n")
    f.write("ncu serialises launches and runs each cold: compare SHARES, not absolute times.\n\n")
    f.write("| id | kernel | us | DRAM read MB | DRAM write MB | GB/s |\n|---|---|---|---|---|---|\n")
    for i, name, t, rd, wr in out_rows:
        f.write(f"| {i} | `{name}` | {t:.1f} | {rd / 1e6:.1f} | {wr / 1e6:.1f} | {(rd + wr) / (t * 1e3) if t else 0:.0f} |\n")
    f.write(f"\nStep total (serialised, cold): {tot:.1f} us\n")
# traffic of the finest-level plane kernels (first dec plane / first interp after tail ...)
dec = [r for r in out_rows if r[1].startswith("k_f3_dec_plane")]
rec = [r for r in out_rows if r[1].startswith("k_f3_rec_plane")]
itp = [r for r in out_rows if r[1].startswith("k_f3_rec_interp")]
if dec:
    traffic["f3_dec_plane@9"] = dec[0][3] + dec[0][4]
if rec:
    traffic["f3_rec_plane@9"] = rec[-1][3] + rec[-1][4]
if itp:
    traffic["f3_rec_interp@9"] = itp[-1][3] + itp[-1][4]
json.dump({"round": rnd, "source": f"profiles/{rnd}_launches.md", "kernels": traffic}, open("profiles/traffic.json", "w"),
          indent=1)
print(open(f"profiles/{rnd}_launches.md").read()[-1500:])
print(traffic)
