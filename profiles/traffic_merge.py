"""DRAM bytes (read + write) of one step's dominant section per configuration, from the ncu launch lists
of profiles/traffic_capture.sh: every launch whose kernel belongs to the section (SpMV / SpMM kernel +
carry fix-up), summed over the one step.  Prints a JSON object keyed like profiles/traffic.json."""
import csv
import json
import sys

SCALE = {"byte": 1.0, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}
SECTION = {"c3": ("spmv+fixup", ("spmv", "fixup")), "c4": ("spmm+fixup", ("spmm", "fixup")),
           "c5": ("spmv+fixup", ("spmv", "fixup"))}
out = {}
for path in sys.argv[1:]:
    cfg = path.rsplit("launches_", 1)[1].split(".")[0]
    sec, pats = SECTION[cfg]
    rows = [r for r in csv.reader(open(path)) if len(r) > 10]
    h = rows[0]
    ik, im, iv, iu = (h.index(c) for c in ("Kernel Name", "Metric Name", "Metric Value", "Metric Unit"))
    tot = 0.0
    for r in rows[1:]:
        name = r[ik].split("(")[0]
        if r[im].startswith("dram__bytes") and any(p in name for p in pats) and "partition" not in name:
            tot += float(r[iv].replace(",", "")) * SCALE.get(r[iu], 1.0)
    out[f"{cfg}:{sec}"] = tot
print(json.dumps(out, indent=1))
