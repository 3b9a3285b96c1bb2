timeout 900 python -m pytest tests -m gpu -x -q -k "combine or dist" > gpurun_out/q_tests.log 2>&1; echo "tests rc=$?"
tail -3 gpurun_out/q_tests.log
timeout 600 python bench.py --no-secondary --no-cpu-baseline --no-e2e > gpurun_out/q_bench.json 2> gpurun_out/q_bench.err; echo "bench rc=$?"
python -c "
import json; d=json.load(open('gpurun_out/q_bench.json')); print(d['ms_per_step'], d['roofline']['frac'], d['roofline']['avg_launch_ms'], d['stage_share'])"
