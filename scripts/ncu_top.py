"""Summarise an ncu report: stall reasons and the hottest SASS lines.
Usage: python scripts/ncu_top.py report.ncu-rep [n] [--kernel REGEX]"""
import csv
import io
import subprocess
import sys

args = [a for a in sys.argv[1:]]
kfilt = []
if "--kernel" in args:
    i = args.index("--kernel")
    kfilt = ["-k", "regex:" + args[i + 1]]
    del args[i:i + 2]
rep = args[0]
n = int(args[1]) if len(args) > 1 else 40
raw = subprocess.run(["ncu", "-i", rep, *kfilt, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
r = list(csv.reader(io.StringIO(raw)))
d = dict(zip(r[0], r[2]))
st = sorted(((k, float(v.replace(",", "") or 0)) for k, v in d.items()
             if "pcsamp_warps_issue_stalled" in k and not k.endswith("not_issued")), key=lambda kv: -kv[1])
tot = sum(v for _, v in st) or 1
print("stalls:", ", ".join(f"{k.split('stalled_')[1]} {v / tot * 100:.1f}%" for k, v in st[:10]))
for k in ["gpu__time_duration.sum", "smsp__inst_executed.sum", "sm__throughput.avg.pct_of_peak_sustained_elapsed",
          "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum", "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum",
          "dram__bytes_read.sum", "dram__bytes_write.sum", "lts__t_sectors_srcunit_tex.sum",
          "smsp__sass_thread_inst_executed_op_ffma_pred_on.sum", "sm__warps_active.avg.pct_of_peak_sustained_active"]:
    if k in d:
        print(f"  {k} = {d[k]}")
src = subprocess.run(["ncu", "-i", rep, *kfilt, "--page", "source", "--csv", "--print-source", "sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(src)))
h = rows[1]
def _num(x):
    try:
        float(x[i_s] or 0)
        return True
    except (ValueError, IndexError):
        return False


data = None
i_s = h.index("Warp Stall Sampling (All Samples)")
data = [x for x in rows[2:] if _num(x)]
i_src = h.index("Source")
i_ex = h.index("Instructions Executed")
tot = sum(float(x[i_s] or 0) for x in data) or 1
for x in sorted(data, key=lambda x: -float(x[i_s] or 0))[:n]:
    print(x[0][-5:], f"{float(x[i_s]) / tot * 100:5.1f}%", x[i_ex].rjust(10), x[i_src][:100])


def region_breakdown(rows_, lo, hi):
    """Stall reasons summed over SASS lines whose execution count is in [lo, hi)."""
    h_ = rows_[1]
    cols = [c for c in h_ if c.startswith("stall_") and "Not Issued" not in c]
    idx = {c: h_.index(c) for c in cols}
    i_e = h_.index("Instructions Executed")
    tot_ = {c: 0.0 for c in cols}
    n_inst = 0
    for x in rows_[2:]:
        e = float(x[i_e] or 0)
        if lo <= e < hi:
            n_inst += 1
            for c in cols:
                tot_[c] += float(x[idx[c]] or 0)
    s_ = sum(tot_.values()) or 1
    return n_inst, {c: round(v / s_ * 100, 1) for c, v in sorted(tot_.items(), key=lambda kv: -kv[1]) if v}


if len(args) > 3:
    print(region_breakdown(rows, float(args[2]), float(args[3])))
