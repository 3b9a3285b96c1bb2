# ncu --set full of every merge kernel of one C5 sort_and_combine (probe_c5, 4th call)
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
timeout 300 ncu -f --set full --clock-control none --import-source on -k regex:"k_" -s 36 -c 18 -o /tmp/c5 python tools/gpu/probe_c5.py > gpurun_out/c5_ncu.log 2>&1; echo "ncu rc=$?"
ncu -i /tmp/c5.ncu-rep --page raw --csv > gpurun_out/c5_raw.csv 2>&1
ncu -i /tmp/c5.ncu-rep --page source --csv --print-source cuda,sass > gpurun_out/c5_src.csv 2>&1
ls -la gpurun_out/c5_* | awk '{print $5, $9}'
