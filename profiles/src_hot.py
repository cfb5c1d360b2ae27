"""Per-source-line totals (instructions executed, stall samples) of one kernel in an .ncu-rep.

usage: python profiles/src_hot.py report.ncu-rep [top_n]
Reads `ncu -i --page source --csv --print-source=cuda,sass` and sums the SASS rows under each CUDA
source line (every file of the kernel)."""
import csv, io, subprocess, sys

rep = sys.argv[1]
top = int(sys.argv[2]) if len(sys.argv) > 2 else 40
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source=cuda,sass"],
                     capture_output=True, text=True).stdout
tot = {}
fname = "?"
hdr = None
for row in csv.reader(io.StringIO(out)):
    if not row:
        continue
    if row[0] == "File Path":
        fname = row[1].split("/")[-1]
        continue
    if row[0] == "Line No":
        hdr = row
        continue
    if hdr is None or row[0] in ("Function Name",) or row[0] == "":
        continue
    try:
        ie = int(row[hdr.index("Instructions Executed")] or 0)
        st = int(row[hdr.index("Warp Stall Sampling (All Samples)")] or 0)
    except (ValueError, IndexError):
        continue
    key = (fname, int(row[0]), row[1][:90])
    a = tot.setdefault(key, [0, 0])
    a[0] += ie
    a[1] += st
T = sum(v[0] for v in tot.values()) or 1
S = sum(v[1] for v in tot.values()) or 1
print(f"total instructions {T}, stall samples {S}")
for (f, ln, src), (ie, st) in sorted(tot.items(), key=lambda t: -t[1][0])[:top]:
    print(f"{ie / T * 100:5.1f}% {st / S * 100:5.1f}%  {f}:{ln}  {src.strip()}")
