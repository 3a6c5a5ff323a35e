# ncu captures of the small-batch merged-stream kernel (k_fc_j) at B = 1 on
# C5 fc6 and C2 fc6: each command first runs plain (exit 0), then under ncu.
set -x
P=gpurun_out/${PJ:-pj}
mkdir -p $P
timeout 600 python -m pytest tests/test_gpu_joint.py -x -q -p no:cacheprovider > $P/test_joint.log 2>&1
for cl in "C5 0" "C2 0" "C5 1" "C5 2"; do
  set -- $cl
  C="python scripts/j_one.py $1 $2 1 2 3"
  timeout 300 $C > $P/plain_j_$1_$2.log 2>&1 || continue
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_fc_j -s 2 -c 1 -f \
    -o $P/j_$1_$2 $C > $P/ncu_j_$1_$2.log 2>&1
  CDN_J_TRACE=$P/jtrace_$1_$2.bin python scripts/j_one.py $1 $2 1 2 1 > /dev/null 2>&1
done
