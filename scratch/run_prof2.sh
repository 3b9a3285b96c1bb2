CMD="python bench.py --steps 1 --warmup 3 --no-secondary --no-cpu-baseline --no-e2e"
$CMD > gpurun_out/plain2.log 2>&1 && ncu --set full --clock-control none --import-source on -k regex:k_leaves -s 3 -c 1 -o /tmp/prof_leaves $CMD > gpurun_out/ncu2.log 2>&1
echo "ncu rc=$?"
ncu -i /tmp/prof_leaves.ncu-rep --page raw --csv > gpurun_out/leaves_raw.csv 2>&1
ncu -i /tmp/prof_leaves.ncu-rep --page details --csv > gpurun_out/leaves_details.csv 2>&1
ncu -i /tmp/prof_leaves.ncu-rep --page source --csv --print-source sass > gpurun_out/leaves_source.csv 2>&1
ls -la gpurun_out/
