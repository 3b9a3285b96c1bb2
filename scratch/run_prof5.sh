CMD="python bench.py --steps 1 --warmup 3 --no-secondary --no-cpu-baseline --no-e2e"
$CMD > gpurun_out/plain6.log 2>&1 && ncu --set full --clock-control none --import-source on -k regex:"k_leaves" -s 3 -c 1 -o /tmp/prof5 $CMD > gpurun_out/ncu5.log 2>&1
ncu -i /tmp/prof5.ncu-rep --page raw --csv > gpurun_out/prof5_raw.csv 2>&1
ncu -i /tmp/prof5.ncu-rep --page source --csv --print-source sass > gpurun_out/prof5_src.csv 2>&1
echo done
