# Round-2 measurement run: GPU suite, bench line (N=1), reference arm, launch list,
# ncu --set full of every pipeline kernel of the headline step (with source pages).
# usage: bash tools/gpu/final_r2.sh <tag>
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
TAG=${1:-r2z}
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,driver_version --format=csv > gpurun_out/${TAG}_gpu.txt
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/${TAG}_gpu_tests.log 2>&1; echo "tests rc=$?"; tail -3 gpurun_out/${TAG}_gpu_tests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > gpurun_out/${TAG}_smoke.log 2>&1; tail -1 gpurun_out/${TAG}_smoke.log
timeout 1500 python bench.py --steps 20 --warmup 5 > gpurun_out/${TAG}_bench.json 2> gpurun_out/${TAG}_bench.err; echo "bench rc=$?"
tail -c 400 gpurun_out/${TAG}_bench.err
timeout 900 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/${TAG}_ref.json 2> gpurun_out/${TAG}_ref.err; echo "ref rc=$?"
CMD="python bench.py --steps 1 --warmup 3 --no-secondary --no-cpu-baseline --no-e2e"
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/${TAG}_launches.csv $CMD > /dev/null 2>&1; echo "ncu launches rc=$?"
PCMD="python tools/gpu/probe_step.py 4"
timeout 1200 ncu -f --set full --clock-control none --import-source on -k regex:"k_count|k_scatter|k_split_prep|k_split_count|k_split_bases|k_split_scatter|k_leaf_sort|k_emit|k_sort_ops|k_sample" -s 40 -c 10 -o /tmp/${TAG}_prof $PCMD > gpurun_out/${TAG}_ncu_full.log 2>&1; echo "ncu full rc=$?"
ncu -i /tmp/${TAG}_prof.ncu-rep --page raw --csv > gpurun_out/${TAG}_prof_raw.csv 2>&1
ncu -i /tmp/${TAG}_prof.ncu-rep --page source --csv --print-source cuda,sass > gpurun_out/${TAG}_prof_src.csv 2>&1
ls -la gpurun_out | grep ${TAG} | awk '{print $5, $9}'
