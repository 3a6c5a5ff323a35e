# Small-batch kernel iteration on the GPU box: parity tests of the B <= 4 paths,
# the B = 1 probe (cold per-launch times), CTA traces of k_fc_j.
P=gpurun_out/${PJ:-ji}
mkdir -p $P
timeout 900 python -m pytest tests/test_gpu_joint.py -x -q -p no:cacheprovider > $P/test_joint.log 2>&1
echo "joint tests rc=$?" >> $P/test_joint.log
timeout 300 python scripts/b1_probe.py 8 > $P/b1_probe.json 2> $P/b1_probe.err
for cl in "C5 0" "C2 0" "C5 1" "C5 2"; do
  set -- $cl
  CDN_J_TRACE=$P/jtrace_$1_$2.bin timeout 120 python scripts/j_one.py $1 $2 1 2 1 > /dev/null 2>&1
done
if [ -n "$NCU" ]; then
  for cl in $NCU; do
    L=${cl%_*}; I=${cl#*_}
    timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_fc_j -s 2 -c 1 -f \
      -o $P/j_${L}_$I python scripts/j_one.py $L $I 1 2 3 > $P/ncu_j_${L}_$I.log 2>&1
  done
fi
