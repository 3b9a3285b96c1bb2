python bench.py > gpurun_out/bench2.json 2> gpurun_out/bench2.err; echo "bench rc=$?"
CMD="python bench.py --steps 1 --warmup 3 --no-secondary --no-cpu-baseline --no-e2e"
$CMD > gpurun_out/plain4.log 2>&1 && ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches2.csv $CMD > /dev/null 2>&1
$CMD > gpurun_out/plain5.log 2>&1 && ncu --set full --clock-control none --import-source on -k regex:"k_leaves|k_scatter|k_split|k_count" -s 4 -c 4 -o /tmp/prof4 $CMD > gpurun_out/ncu4.log 2>&1
ncu -i /tmp/prof4.ncu-rep --page raw --csv > gpurun_out/prof4_raw.csv 2>&1
ncu -i /tmp/prof4.ncu-rep --page details --csv > gpurun_out/prof4_details.csv 2>&1
echo done
