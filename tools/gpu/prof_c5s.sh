# ncu --set full (with source) of the C5 sort_and_combine kernels
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
NAME=${1:-c5s}
timeout 900 ncu -f --set full --clock-control none --import-source on -k regex:"k_pack_ops|k_emit|k_or_masks|k_sample|k_leaf_sort|k_scatter" -s 18 -c 6 -o /tmp/$NAME python tools/gpu/probe_c5.py > gpurun_out/${NAME}_ncu.log 2>&1; echo "ncu rc=$?"
ncu -i /tmp/$NAME.ncu-rep --page raw --csv > gpurun_out/${NAME}_raw.csv 2>&1
ncu -i /tmp/$NAME.ncu-rep --page source --csv --print-source cuda,sass > gpurun_out/${NAME}_src.csv 2>&1
ls -la gpurun_out/${NAME}* | awk '{print $5, $9}'
