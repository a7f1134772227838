"""Side-by-side raw ncu metrics of several single-kernel captures (csv from `ncu -i X --page raw --csv`).
usage: ncu_compare.py a.csv b.csv ... [--grep pattern,pattern]"""
import csv, sys
files = [a for a in sys.argv[1:] if not a.startswith("--")]
pats = None
for a in sys.argv[1:]:
    if a.startswith("--grep="):
        pats = a[len("--grep="):].split(",")
cols = []
for f in files:
    rows = list(csv.reader(open(f).read().splitlines()))
    i0 = next(i for i, r in enumerate(rows) if r and r[0] == "ID")
    hdr, units, vals = rows[i0], rows[i0 + 1], rows[i0 + 2]
    cols.append(dict(zip(hdr, zip(vals, units))))
keys = [k for k in cols[0] if all(k in c for c in cols)]
for k in keys:
    if pats and not any(p in k for p in pats):
        continue
    print(f"{k:90s} " + " ".join(f"{c[k][0]:>18s}" for c in cols) + f" {cols[0][k][1]}")
