# ncu --set full of the C4 conv2 / conv3 launches of k_conv_halo (one step)
P=gpurun_out/${PH:-halo}
mkdir -p $P
C="python scripts/step_breakdown.py --cfg C4 --steps 1"
timeout 300 $C > $P/plain.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_conv_halo" -s 4 -c 2 -f -o $P/halo_full $C > $P/ncu_full.log 2>&1
ncu -i $P/halo_full.ncu-rep --page details --csv > $P/halo_full_details.csv 2>/dev/null
