"""Summarise k_fc_j globaltimer traces (env CDN_J_TRACE=file): per launch,
the stamps of every CTA relative to the earliest CTA entry (us).
Events: 0 entry, 1 index loaded + stream copy issued, 2 griddepcontrol.wait
returned, 3 tables + x in shared memory, 4 first unit's bits staged,
5 last unit decoded, 6 CTA done, 7 (thread 0) table copy issued."""
import struct
import sys

import numpy as np

data = open(sys.argv[1], "rb").read()
o, k = 0, 0
while o < len(data):
    n = struct.unpack_from("<Q", data, o)[0]
    o += 8
    t = np.frombuffer(data, dtype=np.uint64, count=n, offset=o).astype(np.float64).reshape(-1, 8)
    o += 8 * n
    t0 = t[:, 0].min()
    rel = (t - t0) / 1e3
    rel[t == 0] = np.nan
    print(f"launch {k}: {t.shape[0]} CTAs")
    for ev in range(8):
        c = rel[:, ev]
        print(f"  ev{ev}: min {np.nanmin(c):7.2f} med {np.nanmedian(c):7.2f} max {np.nanmax(c):7.2f} us")
    k += 1

# per-CTA phase durations of the last launch (us): staging (entry -> tables
# and x resident), warp 0's decode (ev4 -> ev5), and its wait for the CTA's
# other warps (ev5 -> ev6); CTA entry times show the waves
if k:
    d = lambda a, b: rel[:, b] - rel[:, a]
    for name, a, b in (("staging", 0, 3), ("warp0 decode", 4, 5), ("tail", 5, 6), ("cta", 0, 6)):
        c = d(a, b)
        print(f"  {name:13s}: min {np.nanmin(c):7.2f} med {np.nanmedian(c):7.2f} max {np.nanmax(c):7.2f} us")
    st = np.sort(rel[:, 0])
    print("  entry times (every 16th CTA):", " ".join(f"{v:.1f}" for v in st[::16]))
