# ncu --set full of the dense-bitmatrix kernels (tensor and direct), n=500 M=65536
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
for K in k_bitmatrix_tc k_bitmatrix_direct; do
  timeout 600 ncu -f --set full --clock-control none -k regex:"$K" -c 1 -o /tmp/$K python tools/gpu/probe_bm_dense.py 65536 > gpurun_out/${K}_ncu.log 2>&1; echo "$K rc=$?"
  ncu -i /tmp/$K.ncu-rep --page raw --csv > gpurun_out/${K}_raw.csv 2>&1
done
