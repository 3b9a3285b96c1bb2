nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 900 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err; echo "bench rc=$?"
CMD="python bench.py --steps 1 --warmup 3 --no-secondary --no-cpu-baseline --no-e2e"
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv $CMD > /dev/null 2>&1; echo "ncu1 rc=$?"
timeout 900 ncu -f --set full --clock-control none --import-source on -k regex:"k_leaf_sort|k_emit|k_scatter|k_split_scatter" -s 12 -c 4 -o /tmp/prof $CMD > gpurun_out/ncu_full.log 2>&1; echo "ncu2 rc=$?"
ncu -i /tmp/prof.ncu-rep --page raw --csv > gpurun_out/prof_raw.csv 2>&1
ncu -i /tmp/prof.ncu-rep --page details --csv > gpurun_out/prof_details.csv 2>&1
ncu -i /tmp/prof.ncu-rep --page source --csv --print-source cuda,sass > gpurun_out/prof_src.csv 2>&1
echo done
