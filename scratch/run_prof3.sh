CMD="python bench.py --steps 1 --warmup 3 --no-secondary --no-cpu-baseline --no-e2e"
$CMD > gpurun_out/plain3.log 2>&1 && ncu --set full --clock-control none --import-source on -k regex:"k_leaves|k_scatter|k_split|k_count" -s 12 -c 4 -o /tmp/prof3 $CMD > gpurun_out/ncu3.log 2>&1
echo "ncu rc=$?"
ncu -i /tmp/prof3.ncu-rep --page details --csv > gpurun_out/prof3_details.csv 2>&1
ncu -i /tmp/prof3.ncu-rep --page raw --csv > gpurun_out/prof3_raw.csv 2>&1
ncu -i /tmp/prof3.ncu-rep --page source --csv --print-source sass -k regex:k_leaves > gpurun_out/prof3_leaves_src.csv 2>&1
ls -la gpurun_out | tail -5
