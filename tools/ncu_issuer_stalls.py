"""Warp-stall samples of the MMA issuer loop from an ncu report's SASS source page.

Usage: python tools/ncu_issuer_stalls.py REPORT.ncu-rep
Exports `ncu -i REPORT --page source --csv --print-source sass`, finds the
span of UTCHMMA instructions, and prints the stall-reason totals of that span
plus every instruction with samples."""
import csv
import io
import subprocess
import sys

out = subprocess.run(["ncu", "-i", sys.argv[1], "--page", "source", "--csv", "--print-source", "sass"],
                     capture_output=True, text=True, check=True).stdout
rows = list(csv.reader(io.StringIO(out)))
hdr, data = rows[1], rows[2:]
ix = {h: i for i, h in enumerate(hdr)}
stalls = [h for h in hdr if h.startswith("stall_") and "Not Issued" not in h]
mma = [i for i, r in enumerate(data) if "UTCHMMA" in r[ix["Source"]]]
lo, hi = mma[0] - 60, mma[-1] + 5
tot = {s: 0 for s in stalls}
lines = []
for r in data[lo:hi]:
    n = int(r[ix["Warp Stall Sampling (All Samples)"]] or 0)
    for s in stalls:
        tot[s] += int(r[ix[s]] or 0)
    if n > 0:
        top = sorted(((int(r[ix[s]] or 0), s) for s in stalls), reverse=True)[:2]
        lines.append(f"{r[ix['Source']][:64]:64s} samples {n:4d} exec {r[ix['Instructions Executed']]:>7s} {top}")
print(f"{len(mma)} UTCHMMA sites; stall totals over the issuer span:")
for s, v in sorted(tot.items(), key=lambda x: -x[1])[:10]:
    print(f"  {s:24s} {v}")
print("\n".join(lines))
