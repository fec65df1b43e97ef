"""Per-region warp-stall breakdown of an ncu --set full capture (source page,
SASS).  Regions are split at the warp-role branches by instruction count."""
import csv
import subprocess
import sys


def load(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                         capture_output=True, text=True).stdout
    rows = list(csv.reader(out.splitlines()))
    return rows[1], rows[2:]


def main():
    hdr, data = load(sys.argv[1])
    ia, isrc, isamp, inst = (hdr.index(k) for k in ("Address", "Source",
                                                     "Warp Stall Sampling (All Samples)",
                                                     "Instructions Executed"))
    reasons = [h for h in hdr if h.startswith("stall_") and "Not Issued" not in h]
    ridx = [hdr.index(h) for h in reasons]
    tot = sum(float(r[isamp] or 0) for r in data)
    win = int(sys.argv[2]) if len(sys.argv) > 2 else 48
    for w in range(0, len(data), win):
        chunk = data[w:w + win]
        s = sum(float(r[isamp] or 0) for r in chunk)
        if s / tot < 0.01:
            continue
        agg = [sum(float(r[i] or 0) for r in chunk) for i in ridx]
        top = sorted(zip(reasons, agg), key=lambda x: -x[1])[:4]
        ops = sorted({r[isrc].split()[0] if not r[isrc].startswith("@") else r[isrc].split()[1]
                      for r in chunk if r[isrc].split()})
        key = [o for o in ops if any(k in o for k in ("SYNCS", "LDGSTS", "UTCHMMA", "LDTM", "UTMA",
                                                      "BAR", "DEPBAR", "LDS", "STS", "LDG", "VOTE"))]
        mx = max(float(r[inst] or 0) for r in chunk)
        print(f"{int(chunk[0][ia], 16) & 0xfffff:05x} {100 * s / tot:5.1f}% exec {mx:9.0f} "
              + " ".join(f"{k[6:]}={100 * v / max(s, 1):.0f}" for k, v in top) + f"  {key}")


if __name__ == "__main__":
    main()
