"""Print the SASS lines of an ncu report with the most executed instructions
and warp-stall samples.  usage: python tools/ncu_sass_hot.py rep.ncu-rep [frac]"""
import csv
import io
import subprocess
import sys

rep = sys.argv[1]
frac = float(sys.argv[2]) if len(sys.argv) > 2 else 0.003
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
h = rows[1]
ia, isrc = h.index("Address"), h.index("Source")
iex, ist = h.index("Instructions Executed"), h.index("Warp Stall Sampling (All Samples)")
tot = 0
lines = []
for r in rows[2:]:
    if len(r) <= iex:
        continue
    try:
        n = int(r[iex])
    except ValueError:
        continue
    tot += n
    lines.append((r[ia][-5:], r[isrc].strip(), n, int(r[ist] or 0)))
stall_tot = sum(l[3] for l in lines)
print(f"total executed warp instructions {tot/1e6:.1f}M, stall samples {stall_tot}")
for a, s, n, st in lines:
    if n > tot * frac or st > stall_tot * 0.01:
        print(f"{a} {n/1e6:8.2f}M {st:6d} {s}")
