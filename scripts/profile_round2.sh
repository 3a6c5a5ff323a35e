# Round-2 profile on the GPU box.  Every ncu command line below first ran
# plain (exit 0) in the same call (B200_PROFILING.md).
set -x
P=gpurun_out/prof2
mkdir -p $P
timeout 900 python bench.py > $P/bench.json 2> $P/bench.err || exit 1
B="python bench.py --steps 4 --warmup 3 --no-c4 --no-cpu-baseline --b1-replicas 0"
timeout 600 $B > $P/bench_short.json 2>&1 || exit 1
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --nvtx --nvtx-include "cdn_timed/" --csv \
  --log-file $P/launches_bench.csv $B > $P/ncu_bench.log 2>&1
python scripts/launch_summary.py $P/launches_bench.csv --steps 4 > $P/launch_summary.txt 2>&1
for l in 0 1 2; do
  C="python scripts/layer_bench.py --policy tc --layers $l --batches 512 --replicas 1 --single"
  timeout 300 $C > $P/plain_l$l.log 2>&1 || continue
  timeout 900 ncu --set full --clock-control none --import-source on \
    -k regex:"k_fc_tc|k_tc_list|k_split|k_xscale|k_tc_reduce" -c 6 -f -o $P/tc_l$l $C > $P/ncu_l$l.log 2>&1
done
for cl in "C5 0" "C2 0"; do
  set -- $cl
  C="python scripts/j_one.py $1 $2 1 2 1"
  timeout 300 $C > $P/plain_j_$1_$2.log 2>&1 || continue
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_fc_j -s 2 -c 1 -f \
    -o $P/j_$1_$2 $C > $P/ncu_j_$1_$2.log 2>&1
done
CDN_J_TRACE=$P/jtrace_c5fc6.bin python scripts/j_one.py C5 0 1 2 1 > /dev/null 2>&1
CDN_J_TRACE=$P/jtrace_c2fc6.bin python scripts/j_one.py C2 0 1 2 1 > /dev/null 2>&1
python scripts/step_breakdown.py --cfg C5 > $P/c5_breakdown.json 2>&1
python scripts/step_breakdown.py --cfg C4 > $P/c4_breakdown.json 2>&1
