# ncu --set full of the given kernels in one C4 step (probe_step), CSV pages to gpurun_out/
# usage: bash tools/gpu/prof_r2.sh <regex> <name> [count] [config]
RE="$1"; NAME="$2"; CNT="${3:-4}"; CFG="${4:-4}"
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
CMD="python tools/gpu/probe_step.py $CFG"
$CMD > gpurun_out/${NAME}_plain.log 2>&1 || { echo "plain run failed"; exit 1; }
tail -2 gpurun_out/${NAME}_plain.log
timeout 1200 ncu -f --set full --clock-control none --import-source on -k regex:"$RE" -c $CNT -o /tmp/$NAME $CMD > gpurun_out/${NAME}_ncu.log 2>&1; echo "ncu rc=$?"
ncu -i /tmp/$NAME.ncu-rep --page raw --csv > gpurun_out/${NAME}_raw.csv 2>&1
ncu -i /tmp/$NAME.ncu-rep --page details --csv > gpurun_out/${NAME}_details.csv 2>&1
ncu -i /tmp/$NAME.ncu-rep --page source --csv --print-source cuda,sass > gpurun_out/${NAME}_src.csv 2>&1
ls -la gpurun_out/${NAME}* | awk '{print $5, $9}'
