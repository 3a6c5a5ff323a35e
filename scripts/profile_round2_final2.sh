# Round-2 closing evidence on the GPU box (B200_PROFILING.md: every ncu command line
# first ran plain, exit 0, in the same call).  Output: gpurun_out/$PF
set -x
P=gpurun_out/${PF:-pf2}
mkdir -p $P
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv > $P/smi.txt
timeout 1500 python -m pytest tests -m gpu -x -q -p no:cacheprovider > $P/gpu_tests.log 2>&1; echo "rc=$?" >> $P/gpu_tests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $P/smoke.log 2>&1
timeout 900 python bench.py > $P/bench.json 2> $P/bench.err
B="python bench.py --steps 4 --warmup 3 --no-c4 --no-cpu-baseline --b1-replicas 0"
timeout 600 $B > $P/bench_short.json 2>&1 && \
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --nvtx --nvtx-include "cdn_timed/" --csv \
  --log-file $P/launches_bench.csv $B > $P/ncu_bench.log 2>&1
python scripts/launch_summary.py $P/launches_bench.csv --steps 4 > $P/launch_summary.txt 2>&1
# C4 (AlexNet, B = 64): launch list of six infer calls, then ncu --set full of the last call's CONV-path kernels
C="python scripts/c4_once.py"
timeout 300 $C > $P/plain_c4.log 2>&1 && \
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $P/c4_launches.csv $C > $P/ncu_c4_list.log 2>&1
python scripts/ncu_tail_table.py $P/c4_launches.csv --calls 6 > $P/c4_launch_table.txt 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_conv_halo|k_lrn_pool_rows|k_pool8|k_decode_conv|k_s2d" -s 70 -c 14 -f \
  -o $P/conv_c4 $C > $P/ncu_c4.log 2>&1
for l in 0 1 2; do
  C="python scripts/layer_bench.py --policy tc --layers $l --batches 512 --replicas 1 --single"
  timeout 300 $C > $P/plain_l$l.log 2>&1 && \
  timeout 900 ncu --set full --clock-control none --import-source on \
    -k regex:"k_fc_tc|k_tc_list|k_split|k_xscale|k_tc_reduce" -c 6 -f -o $P/tc_l$l $C > $P/ncu_l$l.log 2>&1
done
for cl in "C5 0" "C2 0"; do
  set -- $cl
  C="python scripts/j_one.py $1 $2 1 2 3"
  timeout 300 $C > $P/plain_j_$1_$2.log 2>&1 && \
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_fc_j -s 2 -c 1 -f \
    -o $P/j_$1_$2 $C > $P/ncu_j_$1_$2.log 2>&1
done
timeout 300 python scripts/step_breakdown.py --cfg C5 > $P/c5_breakdown.json 2>&1
timeout 300 python scripts/step_breakdown.py --cfg C4 > $P/c4_breakdown.json 2>&1
timeout 900 python scripts/grid_report.py > $P/grid.jsonl 2> $P/grid.err
timeout 1200 python scripts/variable_batch_gain.py > $P/variable_batch_c4.jsonl 2> $P/variable_batch.err
