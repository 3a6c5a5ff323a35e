# conv GEMM filter-tile width sweep on C4 (per-layer ncu durations of k_gemm_bf16)
P=gpurun_out/${PB:-bn}
mkdir -p $P
for bn in 256 128 96 64; do
  CDN_GEMM_BN=$bn timeout 300 python scripts/step_breakdown.py --cfg C4 > $P/c4_bn$bn.json 2>&1
  CDN_GEMM_BN=$bn timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:k_gemm_bf16 --csv \
    --log-file $P/launches_bn$bn.csv python scripts/step_breakdown.py --cfg C4 --steps 1 > /dev/null 2>&1
done
