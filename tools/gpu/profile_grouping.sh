# ncu --set full of the K6 resolver on config 3 (batches 10..11)
python tools/gpu/probe_c3.py > gpurun_out/grp_plain.log 2>&1 || exit 1
timeout 900 ncu -f --set full --clock-control none --import-source on -k regex:"k_group_resolve" -s 10 -c 2 -o /tmp/grp python tools/gpu/probe_c3.py > gpurun_out/grp_ncu.log 2>&1; echo "ncu rc=$?"
ncu -i /tmp/grp.ncu-rep --page raw --csv > gpurun_out/grp_raw.csv 2>&1
ncu -i /tmp/grp.ncu-rep --page source --csv --print-source cuda,sass > gpurun_out/grp_src.csv 2>&1
