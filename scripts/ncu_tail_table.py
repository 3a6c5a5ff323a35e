"""Per-kernel table of the LAST `--frac` of an ncu launch list (gpu__time_duration.sum,
--clock-control none): launches, mean / total us by kernel name -- the steady-state
steps of a script that repeats one infer call (warm-up and autotune launches come first)."""
import csv, sys, argparse, collections, re
ap = argparse.ArgumentParser()
ap.add_argument("csv")
ap.add_argument("--calls", type=int, default=1, help="infer calls covered by the tail")
ap.add_argument("--tail", type=int, default=0, help="number of trailing launches to keep (0: all)")
a = ap.parse_args()
rows = []
with open(a.csv, newline="") as f:
    lines = [l for l in f if not l.startswith("==")]
r = csv.DictReader(lines)
for row in r:
    if row.get("Metric Name") != "gpu__time_duration.sum":
        continue
    v = float(row["Metric Value"].replace(",", ""))
    u = row["Metric Unit"]
    v = v / 1e3 if u in ("nsecond", "ns") else v * 1e3 if u in ("msecond", "ms") else v
    rows.append((re.sub(r"\(.*", "", row["Kernel Name"]), v))
if a.tail:
    rows = rows[-a.tail:]
agg = collections.OrderedDict()
for k, v in rows:
    agg.setdefault(k, []).append(v)
tot = sum(v for _, v in rows)
print(f"{len(rows)} launches, {tot / a.calls:.1f} us per call (serialised, cold caches)")
for k, vs in agg.items():
    print(f"{k:40s} n/call {len(vs) / a.calls:5.1f}  mean {sum(vs) / len(vs):8.1f} us  per call {sum(vs) / a.calls:8.1f} us")
