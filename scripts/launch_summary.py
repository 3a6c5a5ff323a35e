"""Summarise an ncu launch list (--metrics gpu__time_duration.sum --csv):
per-kernel launch count, total and mean device time, share of our kernels.
Usage: python scripts/launch_summary.py launches.csv"""
import csv
import re
import sys
from collections import defaultdict

rows = [r for r in csv.reader(open(sys.argv[1])) if len(r) > 10 and r[0] != "ID"]
tot = defaultdict(float)
cnt = defaultdict(int)
grids = defaultdict(set)
for r in rows:
    name = r[4]
    m = re.search(r"(k_\w+)(<[^>]*>)?", name)
    short = (m.group(1) + (m.group(2) or "")) if m and "cdn" in name else ("torch/other: " + name.split("(")[0][-60:])
    if r[12] != "gpu__time_duration.sum":
        continue
    v = float(r[14].replace(",", ""))
    tot[short] += v
    cnt[short] += 1
    grids[short].add(r[8])
ours = sum(v for k, v in tot.items() if not k.startswith("torch/other"))
print(f"{'kernel':60s} {'launches':>8s} {'total_us':>10s} {'mean_us':>9s} {'share_of_ours':>13s}")
for k, v in sorted(tot.items(), key=lambda kv: -kv[1]):
    share = f"{v / ours * 100:12.1f}%" if not k.startswith("torch/other") else ""
    print(f"{k[:60]:60s} {cnt[k]:8d} {v / 1e3:10.1f} {v / cnt[k] / 1e3:9.2f} {share}")
