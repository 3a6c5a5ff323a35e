# k_conv_halo bring-up on the GPU box: per-layer conv parity vs the oracle with
# the halo kernel (descriptor base offset 0, then (addr >> 7) & 7), then C4 timing
# halo vs the im2col-TMA GEMM.
P=gpurun_out/${PH:-halo}
mkdir -p $P
for m in 1 2; do
  CDN_CONV_HALO=$m timeout 600 python -m pytest tests/test_gpu_conv.py -x -q -p no:cacheprovider \
    -k "alexnet_conv_layer_vs_oracle or c4_alexnet_end_to_end" > $P/conv_m$m.log 2>&1
  echo "rc=$?" >> $P/conv_m$m.log
done
for m in 0 1 2; do
  CDN_CONV_HALO=$m timeout 300 python scripts/c4_once.py > $P/c4_m$m.log 2>&1
done
