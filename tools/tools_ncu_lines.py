"""Summarise an `ncu --page source --csv --print-source cuda,sass` dump:
per source line, warp-instructions executed and stall samples (top N)."""
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
top = int(sys.argv[2]) if len(sys.argv) > 2 else 30
cur = None
acc = []
hdr = None
for r in rows:
    if not r:
        continue
    if r[0] == "File Path":
        cur = r[1].split("/")[-1]
        continue
    if r[0] == "Line No":
        hdr = r
        continue
    if hdr is None or not r[0].isdigit():
        continue
    d = dict(zip(hdr, r))
    try:
        ins = int(d.get("Instructions Executed", "0") or 0)
        smp = int(d.get("Warp Stall Sampling (All Samples)", "0") or 0)
    except ValueError:
        continue
    acc.append((ins, smp, f"{cur}:{r[0]}", r[1][:90]))
tot_i = sum(a[0] for a in acc) or 1
tot_s = sum(a[1] for a in acc) or 1
print(f"total warp-instr {tot_i:,}  samples {tot_s:,}")
for ins, smp, loc, src in sorted(acc, key=lambda a: -a[1])[:top]:
    print(f"{100*ins/tot_i:5.1f}% ins {100*smp/tot_s:5.1f}% stall  {loc:22s} {src}")
