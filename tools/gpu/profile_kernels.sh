# usage: bash tools/gpu/profile_kernels.sh <kernel-regex> <name> [count]
RE="$1"; NAME="$2"; CNT="${3:-1}"
CMD="python tools/gpu/probe_step.py"
$CMD > gpurun_out/${NAME}_plain.log 2>&1 || { echo "plain run failed"; exit 1; }
timeout 900 ncu -f --set full --clock-control none --import-source on -k regex:"$RE" -s 4 -c $CNT -o /tmp/$NAME $CMD > gpurun_out/${NAME}_ncu.log 2>&1; echo "ncu rc=$?"
ncu -i /tmp/$NAME.ncu-rep --page raw --csv > gpurun_out/${NAME}_raw.csv 2>&1
ncu -i /tmp/$NAME.ncu-rep --page details --csv > gpurun_out/${NAME}_details.csv 2>&1
ncu -i /tmp/$NAME.ncu-rep --page source --csv --print-source cuda,sass > gpurun_out/${NAME}_src.csv 2>&1 || ncu -i /tmp/$NAME.ncu-rep --page source --csv > gpurun_out/${NAME}_src.csv 2>&1
ls -la gpurun_out | tail -5
