# Round profile on the GPU box: bench without ncu first, then the launch list of
# the same bench command, then one `ncu --set full` capture per (kernel, layer).
set -x
mkdir -p gpurun_out/prof
timeout 600 python bench.py --no-c4 > gpurun_out/prof/bench.json 2> gpurun_out/prof/bench.err || exit 1
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv \
  --log-file gpurun_out/prof/launches_bench_all.csv python bench.py --steps 2 --warmup 1 --no-c4 --no-cpu-baseline \
  > gpurun_out/prof/ncu_bench_all.log 2>&1
# the timed region only (NVTX range "cdn_timed" around each timed step)
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --nvtx --nvtx-include "cdn_timed/" --csv \
  --log-file gpurun_out/prof/launches_bench.csv python bench.py --steps 4 --warmup 3 --no-c4 --no-cpu-baseline \
  > gpurun_out/prof/ncu_bench.log 2>&1
for l in 0 1 2; do
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:"k_fc_tc|k_tc_list|k_split_x|k_tc_reduce" -c 4 -f \
    -o gpurun_out/prof/tc_l$l python scripts/layer_bench.py --policy tc --layers $l --batches 512 --replicas 1 --single \
    > gpurun_out/prof/ncu_l$l.log 2>&1
done
python scripts/launch_summary.py gpurun_out/prof/launches_bench.csv --steps 4 > gpurun_out/prof/launch_summary.txt
python scripts/step_breakdown.py --cfg C4 > gpurun_out/prof/c4_breakdown.json 2>&1
python scripts/step_breakdown.py --cfg C5 > gpurun_out/prof/c5_breakdown.json 2>&1
