python tools/gpu/probe_bm.py 3 > gpurun_out/bm_plain.log 2>&1 || exit 1
timeout 900 ncu -f --set full --clock-control none --import-source on -k regex:"k_bitmatrix" -s 1 -c 1 -o /tmp/bm python tools/gpu/probe_bm.py 2 > gpurun_out/bm_ncu.log 2>&1; echo "ncu rc=$?"
ncu -i /tmp/bm.ncu-rep --page raw --csv > gpurun_out/bm_raw.csv 2>&1
ncu -i /tmp/bm.ncu-rep --page source --csv --print-source cuda,sass > gpurun_out/bm_src.csv 2>&1
cat gpurun_out/bm_plain.log
