# k_fc_j parameter sweep at B = 1 (joint LUT width, lanes per row) on C5 fc6 / C2 fc6
P=gpurun_out/${PJ:-jsw}
mkdir -p $P
for jl in 12 13 14; do for jg in 16 32; do
  CDN_JL=$jl CDN_JG=$jg B1_LAYERS=C5:0,C2:0 timeout 300 python scripts/b1_probe.py 8 > $P/jl${jl}_jg${jg}.json 2>&1
done; done
B1_LAYERS=C5:0,C2:0,C5:1,C5:2 CDN_J_MC=1 timeout 300 python scripts/b1_probe.py 8 > $P/mc.json 2>&1
