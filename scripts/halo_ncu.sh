# k_conv_halo on the GPU box: conv parity vs the oracle, then per-launch time,
# tensor-pipe activity and L2 traffic of the C4 conv GEMMs (one step), halo vs
# the im2col-TMA GEMM, and the C4 step time
P=gpurun_out/${PH:-halo}
mkdir -p $P
timeout 600 python -m pytest tests/test_gpu_conv.py -x -q -p no:cacheprovider > $P/conv_tests.log 2>&1
echo "rc=$?" >> $P/conv_tests.log
C="python scripts/step_breakdown.py --cfg C4 --steps 2"
for m in 0 1; do
  export CDN_CONV_HALO=$m
  timeout 300 python scripts/c4_once.py > $P/c4_m$m.log 2>&1
  timeout 300 $C > $P/plain_m$m.log 2>&1 && \
  timeout 600 ncu --clock-control none -k regex:"k_gemm_bf16|k_conv_halo" -s 10 -c 10 --csv \
    --metrics gpu__time_duration.sum,sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed,lts__t_bytes.sum,dram__bytes_read.sum \
    $C > $P/ncu_m$m.csv 2> $P/ncu_m$m.err
done
