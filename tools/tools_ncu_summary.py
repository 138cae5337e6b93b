"""Summarise `ncu --set full` captures (.ncu-rep) into a markdown table:
duration, DRAM bytes, throughputs, issue/occupancy, top stall reasons and
the hottest source lines.  usage: tools_ncu_summary.py out.md a.ncu-rep ..."""
import csv
import io
import subprocess
import sys

csv.field_size_limit(10**9)
sys.path.insert(0, __import__("os").path.dirname(__import__("os").path.abspath(__file__)))
from tools_ncu_csv import SCALE

WANT = [("gpu__time_duration.sum", "duration us", 1e6),
        ("dram__bytes_read.sum", "DRAM read MB", 1e-6),
        ("dram__bytes_write.sum", "DRAM write MB", 1e-6),
        ("dram__throughput.avg.pct_of_peak_sustained_elapsed", "DRAM % peak", 1),
        ("sm__throughput.avg.pct_of_peak_sustained_elapsed", "SM % peak", 1),
        ("smsp__issue_active.avg.pct_of_peak_sustained_active", "issue active %", 1),
        ("sm__warps_active.avg.pct_of_peak_sustained_active", "warps active %", 1),
        ("smsp__inst_executed.sum", "warp instr (M)", 1e-6),
        ("launch__registers_per_thread", "regs", 1),
        ("launch__grid_size", "grid", 1),
        ("launch__block_size", "block", 1)]


def raw(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    vals = {}
    for name, unit, val in zip(rows[0], rows[1], rows[2]):
        try:
            vals[name] = float(val.replace(",", "")) * SCALE.get(unit, 1.0)
        except ValueError:
            vals[name] = val
    return vals


def lines(rep, top=6):
    out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                         capture_output=True, text=True).stdout
    cur, hdr, acc = None, None, []
    for r in csv.reader(io.StringIO(out)):
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
            smp = int(d.get("Warp Stall Sampling (All Samples)", "0") or 0)
        except ValueError:
            continue
        acc.append((smp, f"{cur}:{r[0]}", r[1].strip()[:70]))
    tot = sum(a[0] for a in acc) or 1
    acc.sort(reverse=True)
    return [(100.0 * a[0] / tot, a[1], a[2]) for a in acc[:top]]


def main():
    out, reps = sys.argv[1], sys.argv[2:]
    md = ["# ncu --set full summaries (one launch each, `--clock-control none`)", "",
          "Captured with tools_ncu_full.sh on the B200 box after the same bench command exited 0 without ncu.", ""]
    for rep in reps:
        v = raw(rep)
        name = str(v.get("Kernel Name", rep))
        md.append(f"## `{name[:90]}`")
        md.append("")
        md.append("| metric | value |")
        md.append("|---|---|")
        for key, label, sc in WANT:
            if isinstance(v.get(key), float):
                md.append(f"| {label} | {v[key] * sc:.1f} |")
        st = {k.replace("smsp__pcsamp_warps_issue_stalled_", ""): (x if isinstance(x, float) else 0.0) for k, x in v.items()
              if k.startswith("smsp__pcsamp_warps_issue_stalled_") and not k.endswith("not_issued")}
        tot = sum(st.values()) or 1.0
        top = sorted(st.items(), key=lambda kv: -kv[1])[:6]
        md.append("| top stalls | " + ", ".join(f"{k} {100 * x / tot:.0f}%" for k, x in top) + " |")
        md.append("")
        md.append("Hottest source lines (share of stall samples):")
        md.append("")
        for pct, loc, src in lines(rep):
            md.append(f"* {pct:.1f}% `{loc}` `{src}`")
        md.append("")
    open(out, "w").write("\n".join(md) + "\n")


if __name__ == "__main__":
    main()
