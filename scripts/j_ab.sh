# k_fc_j A/B on the GPU box: joint-kernel parity tests, then the B = 1 cold
# probe and CTA traces with and without the lane-interleaved stream copy.
P=gpurun_out/${PJ:-jab}
mkdir -p $P
timeout 900 python -m pytest tests/test_gpu_joint.py -x -q -p no:cacheprovider > $P/test_joint.log 2>&1
echo "joint tests rc=$?" >> $P/test_joint.log
timeout 300 python scripts/b1_probe.py 8 > $P/b1_probe.json 2> $P/b1_probe.err
CDN_J_NOILV=1 timeout 300 python scripts/b1_probe.py 8 > $P/b1_probe_noilv.json 2> $P/b1_probe_noilv.err
for cl in "C5 0" "C2 0"; do
  set -- $cl
  CDN_J_TRACE=$P/jtrace_$1_$2.bin timeout 120 python scripts/j_one.py $1 $2 1 2 1 > /dev/null 2>&1
done
