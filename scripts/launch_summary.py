"""Summarise an ncu launch list (--metrics gpu__time_duration.sum --csv, with or
without --nvtx columns): per-kernel launch count, total and mean device time,
share of our kernels, and (with --steps N) time per step.
Usage: python scripts/launch_summary.py launches.csv [--steps N]"""
import csv
import re
import sys
from collections import defaultdict

args = sys.argv[1:]
steps = 0
if "--steps" in args:
    i = args.index("--steps")
    steps = int(args[i + 1])
    del args[i:i + 2]
lines = [r for r in csv.reader(open(args[0]))]
hdr_i = next(i for i, r in enumerate(lines) if r and r[0] == "ID")
h = lines[hdr_i]
c_name, c_metric, c_unit, c_val = (h.index("Kernel Name"), h.index("Metric Name"), h.index("Metric Unit"),
                                   h.index("Metric Value"))
scale = {"ns": 1.0, "usecond": 1e3, "us": 1e3, "msecond": 1e6, "ms": 1e6, "nsecond": 1.0}
tot = defaultdict(float)
cnt = defaultdict(int)
for r in lines[hdr_i + 1:]:
    if len(r) <= c_val or r[c_metric] != "gpu__time_duration.sum":
        continue
    name = r[c_name]
    m = re.search(r"(k_\w+)(<[^>]*>)?", name)
    short = (m.group(1) + (m.group(2) or "")) if m else ("torch/other: " + name.split("(")[0][-60:])
    v = float(r[c_val].replace(",", "")) * scale.get(r[c_unit], 1.0)  # ns
    tot[short] += v
    cnt[short] += 1
ours = sum(v for k, v in tot.items() if not k.startswith("torch/other"))
print(f"{'kernel':60s} {'launches':>8s} {'total_us':>10s} {'mean_us':>9s} {'share_of_ours':>13s}"
      + (f" {'us_per_step':>11s}" if steps else ""))
for k, v in sorted(tot.items(), key=lambda kv: -kv[1]):
    share = f"{v / ours * 100:12.1f}%" if not k.startswith("torch/other") else " " * 13
    per = f" {v / steps / 1e3:11.1f}" if steps else ""
    print(f"{k[:60]:60s} {cnt[k]:8d} {v / 1e3:10.1f} {v / cnt[k] / 1e3:9.2f} {share}{per}")
print(f"{'(all ours)':60s} {sum(c for k, c in cnt.items() if not k.startswith('torch')):8d} {ours / 1e3:10.1f}"
      + (f" {'':9s} {'':13s} {ours / steps / 1e3:11.1f}" if steps else ""))
