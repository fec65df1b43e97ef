"""Barrier-wait and top-stall summary of one ncu --set full capture (SASS
source page): every SYNCS try-wait with its execution count (retries) and
stall samples, then the top-N instructions by stall samples.
    python tools/ncu_waits.py <report.ncu-rep> [N]"""
import csv
import subprocess
import sys

rep = sys.argv[1]
top_n = int(sys.argv[2]) if len(sys.argv) > 2 else 20
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(out.splitlines()))
hdr, data = rows[1], rows[2:]
isrc, isamp, iex = (hdr.index(k) for k in ("Source", "Warp Stall Sampling (All Samples)",
                                             "Instructions Executed"))
reasons = [h for h in hdr if h.startswith("stall_") and "Not Issued" not in h]
tot = sum(float(r[isamp] or 0) for r in data)
print(f"total samples {tot:.0f}")
print("-- barrier waits (line, samples incl. next, executions, instruction)")
for i, r in enumerate(data):
    if "TRYWAIT" in r[isrc] and int(r[iex] or 0) > 0:
        s = float(r[isamp] or 0) + float(data[i + 1][isamp] or 0)
        print(f"{i:5d} {s:6.0f} {r[iex]:>9} {r[isrc][:72]}")
print("-- top instructions")
for r in sorted(data, key=lambda r: -float(r[isamp] or 0))[:top_n]:
    rs = sorted(((float(r[hdr.index(h)] or 0), h[6:]) for h in reasons), reverse=True)[:2]
    print(f"{float(r[isamp]) / tot * 100:5.1f}% {r[isrc][:60]:60s} {rs}")
