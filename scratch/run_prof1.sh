python scratch/prof_host.py
CMD="python bench.py --steps 1 --warmup 3 --no-secondary --no-cpu-baseline --no-e2e"
$CMD > gpurun_out/plain2.log 2>&1 && ncu --set full --clock-control none --import-source on -k regex:k_leaves -s 3 -c 1 -o gpurun_out/prof_leaves $CMD > gpurun_out/ncu2.log 2>&1
echo "ncu rc=$?"
