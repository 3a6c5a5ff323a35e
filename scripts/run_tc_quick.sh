# quick TC-path check on the GPU box: TC parity tests, per-layer timing (forced TC), CTA-0 trace of fc6 B=512
timeout 300 python -m pytest tests -m gpu -x -q -k "tc or TC" > gpurun_out/gpu_tc.log 2>&1; tail -3 gpurun_out/gpu_tc.log
timeout 300 python scripts/layer_bench.py --policy tc --batches 128,256,512 > gpurun_out/layer_tc3.log 2>&1
CDN_TC_TRACE=gpurun_out/tc_trace.bin timeout 300 python scripts/layer_bench.py --policy tc --layers 0 --batches 512 --replicas 1 --single > gpurun_out/trace.log 2>&1
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/tc_launches.csv python scripts/layer_bench.py --policy tc --layers 0 --batches 512 --replicas 1 --single > /dev/null 2>&1
