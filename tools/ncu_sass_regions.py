"""Per-region breakdown of an ncu report's SASS page (development tool): groups consecutive
instructions with equal execution counts and prints those above 1 % of instructions or samples."""
import csv
import subprocess
import sys

rep = sys.argv[1]
thr = float(sys.argv[2]) if len(sys.argv) > 2 else 0.01
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source=sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(out.splitlines()))
h = rows[1]
iE, iS, iSrc = h.index("Instructions Executed"), h.index("Warp Stall Sampling (All Samples)"), h.index("Source")
R = rows[2:]
tot = sum(float(r[iE] or 0) for r in R)
totS = sum(float(r[iS] or 0) for r in R)
print(f"total warp instructions {tot:.4g}, samples {totS:.0f}")
segs, cur = [], None
for i, r in enumerate(R):
    e, s = float(r[iE] or 0), float(r[iS] or 0)
    if cur and abs(cur["e"] - e) <= 0.02 * max(cur["e"], 1):
        cur["n"] += 1
        cur["s"] += s
        cur["end"] = i
    else:
        cur = {"e": e, "n": 1, "s": s, "start": i, "end": i}
        segs.append(cur)
for g in segs:
    if g["s"] / totS > thr or g["e"] * g["n"] / tot > thr:
        print(f"[{g['start']:4d}-{g['end']:4d}] n={g['n']:3d} exec/inst={g['e']:.3g} inst%={g['e'] * g['n'] / tot * 100:5.1f} "
              f"samp%={g['s'] / totS * 100:5.1f}  {R[g['start']][iSrc][:60]}")
