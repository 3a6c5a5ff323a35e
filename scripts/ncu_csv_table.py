"""Per-launch table from an `ncu --csv --metrics ...` log: one line per kernel
launch with each metric (usage: python scripts/ncu_csv_table.py FILE...)."""
import collections
import csv
import sys

for f in sys.argv[1:]:
    rows = [r for r in csv.reader(open(f)) if len(r) > 10]
    if not rows:
        print(f, "(no launches)")
        continue
    hdr = rows[0]
    ii, ki, mi, ui, vi = (hdr.index(k) for k in ("ID", "Kernel Name", "Metric Name", "Metric Unit", "Metric Value"))
    d = collections.OrderedDict()
    for r in rows[1:]:
        e = d.setdefault(r[ii], {"kernel": r[ki][:40]})
        e[r[mi]] = (float(r[vi].replace(",", "")), r[ui])
    print(f)
    for k, e in d.items():
        print("  " + e.pop("kernel").ljust(40) + "  " + "  ".join(f"{m.split('.')[0].split('__')[-1]}={v:.4g}{u}" for m, (v, u) in e.items()))
