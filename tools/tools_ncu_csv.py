"""Shared parsing of `ncu --csv` launch lists (unit-aware) and the step
boundary of one bench decompose+recompose step."""
import collections
import csv

SCALE = {"nsecond": 1e-9, "ns": 1e-9, "usecond": 1e-6, "us": 1e-6, "msecond": 1e-3, "ms": 1e-3, "second": 1.0,
         "byte": 1.0, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "Tbyte": 1e12}


def read_launches(path):
    """[(id, kernel, {metric: value in s / bytes})] in launch order."""
    rows = list(csv.reader(open(path)))
    hi = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
    h = rows[hi]
    ki, mi, vi, idi = h.index("Kernel Name"), h.index("Metric Name"), h.index("Metric Value"), h.index("ID")
    ui = h.index("Metric Unit") if "Metric Unit" in h else None
    per = collections.OrderedDict()
    for r in rows[hi + 1:]:
        if len(r) <= vi:
            continue
        sc = SCALE.get(r[ui], 1.0) if ui is not None else 1.0
        per.setdefault((int(r[idi]), r[ki]), {})[r[mi]] = float(r[vi].replace(",", "")) * sc
    return [(i, k, m) for (i, k), m in per.items()]


def short(k):
    return k.split("(")[0].replace("void ", "").replace("mgrx_b200::", "").replace("<unnamed>::", "")


def nbytes(m):
    return m.get("dram__bytes_read.sum", 0.0) + m.get("dram__bytes_write.sum", 0.0)


def last_step(items):
    """Launches of the last step (library kernels only): from the last
    finest-level decompose plane launch (the dec-plane launch moving the most
    bytes) to the end."""
    items = [it for it in items if "mgrx_b200" in it[1] or "k_f3_" in it[1] or "k_tail" in it[1]]
    dec = [n for n, (i, k, m) in enumerate(items) if "dec_plane" in k or "k_dec_coef" in k]
    if not dec:
        return items
    mx = max(nbytes(items[n][2]) for n in dec)
    rec = [n for n, (i, k, m) in enumerate(items) if "rec_plane" in k or "rec_interp" in k or "k_tail_recompose" in k]
    # the last finest-level decompose that a recompose follows, up to the
    # first kernel after that step which belongs to neither (e.g. quantize)
    starts = [n for n in dec if nbytes(items[n][2]) >= 0.5 * mx and rec and rec[-1] > n]
    start = starts[-1] if starts else dec[-1]
    end = len(items)
    for n in range(start + 1, len(items)):
        if "quant" in items[n][1] or (n in dec and nbytes(items[n][2]) >= 0.5 * mx):
            end = n
            break
    return items[start:end]
