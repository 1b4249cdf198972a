"""Top stall reasons of an ncu capture (raw page) and the SASS lines holding
the most warp-state samples (source page).  Diagnostic only.
    python tools/stall_lines.py <raw.csv> <source.csv> [min_share]"""
import csv
import sys

raw, src = sys.argv[1], sys.argv[2]
share = float(sys.argv[3]) if len(sys.argv) > 3 else 0.01
rows = list(csv.reader(open(raw)))
h, v = rows[0], rows[2]
st = [(n, v[i]) for i, n in enumerate(h) if "pcsamp_warps_issue_stalled" in n and not n.endswith("not_issued")]
st = sorted([(n.split("stalled_")[1], float(x)) for n, x in st if x.replace(".", "", 1).isdigit()], key=lambda t: -t[1])
tot = sum(x for _, x in st)
print("stalls:", ", ".join(f"{n} {x / tot:.0%}" for n, x in st[:9]))
rows = list(csv.reader(open(src)))
h, body = rows[1], rows[2:]
si, ie = h.index("Warp Stall Sampling (All Samples)"), h.index("Instructions Executed")
cols = [c for c in h if c.startswith("stall_") and "Not Issued" not in c]
tot = sum(int(r[si]) for r in body if r[si].isdigit())
cum = 0
for k, r in enumerate(body):
    s = int(r[si]) if r[si].isdigit() else 0
    cum += s
    if s >= tot * share:
        top = sorted([(c[6:], int(r[h.index(c)]) if r[h.index(c)].isdigit() else 0) for c in cols], key=lambda t: -t[1])[:2]
        print(f"{k:5d} {s / tot:5.1%} cum {cum / tot:4.0%} x{r[ie]:>8} {r[1].strip()[:64]:64s} {top}")
