"""Print the CTA-0 event timeline of one k_fc_tc launch recorded with
CDN_TC_TRACE=<file> (16 events x 256 slots of %globaltimer ns; 0 = unset),
relative to the CTA start (event 5).  Usage: python scripts/tc_trace_dump.py FILE"""
import sys

import numpy as np

NAMES = {0: "s0 expand begin", 2: "s0 wempty ok", 3: "s0 tile built", 4: "s1 expand begin", 6: "s1 wempty ok",
         7: "s1 tile built", 5: "cta start", 8: "mma wait W", 9: "mma W ok", 10: "mma X ok", 11: "mma issued",
         12: "epi wait", 13: "epi acc ready", 14: "epi done"}
t = np.fromfile(sys.argv[1], dtype=np.uint64).reshape(16, 256).astype(np.int64)
t0 = t[5, 0]
for ev in sorted(NAMES):
    v = t[ev]
    idx = np.nonzero(v)[0]
    if len(idx) == 0:
        continue
    rel = (v[idx] - t0) / 1e3
    head = ", ".join(f"{i}:{r:.2f}" for i, r in zip(idx[:6], rel[:6]))
    tail = ", ".join(f"{i}:{r:.2f}" for i, r in zip(idx[-3:], rel[-3:])) if len(idx) > 6 else ""
    print(f"{NAMES[ev]:16s} n={len(idx):3d}  us: {head}{' ... ' + tail if tail else ''}")
