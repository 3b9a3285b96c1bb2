set -x
python bench.py > gpurun_out/bench1.json 2> gpurun_out/bench1.err
echo "bench rc=$?"
tail -3 gpurun_out/bench1.err
CMD="python bench.py --steps 2 --warmup 3 --no-secondary --no-cpu-baseline --no-e2e"
$CMD > gpurun_out/plain.log 2>&1 && ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv $CMD > gpurun_out/ncu.log 2>&1
echo "ncu rc=$?"
