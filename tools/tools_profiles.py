"""Turn an ncu launch list (gpu__time_duration + dram bytes) into the
committed per-round summary: profiles/<round>_launches.md and
profiles/traffic.json (DRAM bytes per launch of each kernel@level, used by
bench.py for roofline.traffic).  Kernel@level is recovered from launch order
of one decompose+recompose step (the last one in the list)."""
import collections
import csv
import json
import sys

import os

sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
from tools_ncu_csv import last_step, read_launches, short  # noqa: E402

src, rnd = sys.argv[1], sys.argv[2]
step = last_step(read_launches(src))
out_rows = []
traffic = {}
for i, k, m in step:
    t = m.get("gpu__time_duration.sum", 0) * 1e6
    out_rows.append((i, short(k), t, m.get("dram__bytes_read.sum", 0), m.get("dram__bytes_write.sum", 0)))
tot = sum(r[2] for r in out_rows)
with open(f"profiles/{rnd}_launches.md", "w") as f:
    f.write(f"# {rnd}: ncu launch list, one decompose + recompose step of the 513^3 fp32 bench\n\n")
    f.write("Command: `ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum "
            "--clock-control none --csv python tools/tools_step.py` (tools/tools_prof.sh: two eager decompose + "
            "recompose steps of the bench field; the last step is listed).\n")
    f.write("ncu serialises launches and runs each cold: compare SHARES, not absolute times.\n\n")
    f.write("| id | kernel | us | DRAM read MB | DRAM write MB | GB/s |\n|---|---|---|---|---|---|\n")
    for i, name, t, rd, wr in out_rows:
        f.write(f"| {i} | `{name}` | {t:.1f} | {rd / 1e6:.1f} | {wr / 1e6:.1f} | {(rd + wr) / (t * 1e3) if t else 0:.0f} |\n")
    f.write(f"\nStep total (serialised, cold): {tot:.1f} us\n")
# traffic of the finest-level plane kernels (first dec plane / first interp after tail ...)
dec = [r for r in out_rows if r[1].startswith("k_f3_dec_plane")]
rec = [r for r in out_rows if r[1].startswith("k_f3_rec_plane")]
itp = [r for r in out_rows if r[1].startswith("k_f3_rec_interp")]
# the finest level's launch of each kind moves the most bytes
for tag, rows_ in (("f3_dec_plane@9", dec), ("f3_rec_plane@9", rec), ("f3_rec_interp@9", itp)):
    if rows_:
        r = max(rows_, key=lambda r: r[3] + r[4])
        traffic[tag] = r[3] + r[4]
step_bytes = sum(r[3] + r[4] for r in out_rows)
with open(f"profiles/{rnd}_launches.md", "a") as f:
    f.write(f"Step DRAM traffic (all kernels): {step_bytes / 1e9:.3f} GB (algorithmic 2.471 GB)\n")
json.dump({"round": rnd, "source": f"profiles/{rnd}_launches.md", "kernels": traffic, "step": step_bytes},
          open("profiles/traffic.json", "w"), indent=1)
print(open(f"profiles/{rnd}_launches.md").read()[-1500:])
print(traffic)
