"""Record the DRAM traffic of one kernel launch from an `ncu --set full`
report into profiles/traffic.json (read by bench.py for roofline.traffic).
Usage: python scripts/traffic_from_ncu.py REPORT.ncu-rep "KERNEL LABEL" [KERNEL_REGEX]"""
import csv
import io
import json
import os
import subprocess
import sys

rep, label = sys.argv[1], sys.argv[2]
kf = ["-k", "regex:" + sys.argv[3]] if len(sys.argv) > 3 else []
raw = subprocess.run(["ncu", "-i", rep, *kf, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
r = list(csv.reader(io.StringIO(raw)))
h, units, vals = r[0], r[1], r[2]
scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}


def get(k):
    i = h.index(k)
    return float(vals[i].replace(",", "")) * scale[units[i]]


tot = get("dram__bytes_read.sum") + get("dram__bytes_write.sum")
path = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "profiles", "traffic.json")
d = json.load(open(path)) if os.path.exists(path) else {}
d[label] = {"dram_bytes": tot, "source": os.path.basename(rep),
            "duration_under_ncu": (vals[h.index("gpu__time_duration.sum")] + " " + units[h.index("gpu__time_duration.sum")])
            if "gpu__time_duration.sum" in h else None}
json.dump(d, open(path, "w"), indent=1)
print(label, tot)
