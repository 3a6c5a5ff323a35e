"""Copy one closing-evidence run (scripts/profile_round2_final2.sh, gpurun_out/<dir>) into
profiles/ under the round's names and derive the text summaries from the ncu reports.
Usage: python scripts/collect_round2.py gpurun_out/pf2"""
import csv
import io
import os
import shutil
import subprocess
import sys

src = sys.argv[1]
dst = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "profiles")


def cp(a, b):
    pa = os.path.join(src, a)
    if os.path.exists(pa) and os.path.getsize(pa) > 0:
        shutil.copyfile(pa, os.path.join(dst, b))
        print("copied", a, "->", b)
    else:
        print("MISSING", a)


def last_json_line(a, b):
    pa = os.path.join(src, a)
    if not os.path.exists(pa):
        print("MISSING", a)
        return
    lines = [l for l in open(pa).read().splitlines() if l.startswith("{")]
    if lines:
        open(os.path.join(dst, b), "w").write(lines[-1] + "\n")
        print("copied", a, "->", b)


def raw_rows(rep):
    raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    r = list(csv.reader(io.StringIO(raw)))
    return [dict(zip(r[0], row)) for row in r[2:]] if len(r) > 2 else []


def conv_table(rep, out, title):
    rows = raw_rows(rep)
    with open(out, "w") as f:
        f.write(f"# {title}\n# kernel | us | tensor pipe % of peak (sm__pipe_tensor_cycles_active) | issue active % | XU pipe % | "
                "DRAM read MB | DRAM write MB | grid x block | warps active %\n")
        for d in rows:
            def g(k):
                return next((d[x] for x in d if x.startswith(k)), "")
            f.write(" | ".join([d.get("Kernel Name", "")[:44], g("gpu__time_duration.sum"),
                                g("sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed") or
                                g("sm__pipe_tensor_subpipe_hmma_cycles_active"),
                                g("smsp__issue_active.avg.pct_of_peak_sustained_active"),
                                g("sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active"),
                                g("dram__bytes_read.sum"), g("dram__bytes_write.sum"),
                                g("launch__grid_size") + "x" + g("launch__block_size"),
                                g("sm__warps_active.avg.pct_of_peak_sustained_active")]) + "\n")
    print("wrote", out)


def top(rep, kernel, out):
    here = os.path.dirname(os.path.abspath(__file__))
    r = subprocess.run([sys.executable, os.path.join(here, "ncu_top.py"), rep, "40", "--kernel", kernel],
                       capture_output=True, text=True)
    open(out, "w").write(r.stdout)
    print("wrote", out)


cp("gpu_tests.log", "r02_gpu_tests.log")
last_json_line("bench.json", "r02_bench.json")
cp("launches_bench.csv", "r02_launches_bench.csv")
cp("launch_summary.txt", "r02_launch_summary.txt")
cp("c4_launches.csv", "r02_c4_launches.csv")
cp("c4_launch_table.txt", "r02_c4_launch_table.txt")
last_json_line("c5_breakdown.json", "r02_c5_step_breakdown.json")
last_json_line("c4_breakdown.json", "r02_c4_step_breakdown.json")
cp("grid.jsonl", "r02_grid.jsonl")
cp("variable_batch_c4.jsonl", "r02_variable_batch_c4.jsonl")
cp("conv_c4.ncu-rep", "r02_conv_c4_b64.ncu-rep")
if os.path.exists(os.path.join(dst, "r02_conv_c4_b64.ncu-rep")):
    conv_table(os.path.join(dst, "r02_conv_c4_b64.ncu-rep"), os.path.join(dst, "r02_conv_c4_b64_summary.txt"),
               "C4 AlexNet B = 64 CONV-path kernels of one infer call, ncu --set full --clock-control none: k_decode_conv "
               "(side stream), k_s2d, k_conv_halo per layer, k_lrn_pool_rows, k_pool8")
for l, name in ((0, "fc6"), (1, "fc7"), (2, "fc8")):
    cp(f"tc_l{l}.ncu-rep", f"r02_tc_path_{name}_b512.ncu-rep")
    rep = os.path.join(dst, f"r02_tc_path_{name}_b512.ncu-rep")
    if os.path.exists(rep):
        for k, tag in (("k_fc_tc", "k_fc_tc"), ("k_tc_list", "k_tc_list"), ("k_split|k_scale_split", "k_split"),
                       ("k_tc_reduce", "k_tc_reduce")):
            top(rep, k, os.path.join(dst, f"r02_{tag}_{name}_b512_summary.txt"))
for cfg in ("C5", "C2"):
    cp(f"j_{cfg}_0.ncu-rep", f"r02_k_fc_j_{cfg}_fc6_b1.ncu-rep")
    rep = os.path.join(dst, f"r02_k_fc_j_{cfg}_fc6_b1.ncu-rep")
    if os.path.exists(rep):
        top(rep, "k_fc_j", os.path.join(dst, f"r02_k_fc_j_{cfg}_fc6_b1_summary.txt"))
