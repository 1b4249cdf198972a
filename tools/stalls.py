"""Top SASS instructions by warp-stall samples from an ncu report (source page).

    python tools/stalls.py <report.ncu-rep> [N]
"""
import csv
import subprocess
import sys

rep = sys.argv[1]
n = int(sys.argv[2]) if len(sys.argv) > 2 else 40
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(out.splitlines()))
hdr = next(r for r in rows if "Address" in r and "Source" in r)
body = [r for r in rows[rows.index(hdr) + 1:] if len(r) == len(hdr)]
ia, isrc = hdr.index("Address"), hdr.index("Source")
iall = hdr.index("Warp Stall Sampling (All Samples)")
ini = hdr.index("Warp Stall Sampling (Not-issued Samples)")
tot = sum(float(r[iall] or 0) for r in body) or 1.0
print(f"total stall samples {tot:.0f}")
for k, r in sorted(enumerate(body), key=lambda kr: -float(kr[1][iall] or 0))[:n]:
    print(f"{100 * float(r[iall]) / tot:5.1f}% {r[ini]:>7} #{k:5d} {r[isrc].strip()[:110]}")
