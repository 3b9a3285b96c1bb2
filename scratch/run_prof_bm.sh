python scratch/quick_bm.py > gpurun_out/bm_plain.log 2>&1 && ncu --set full --clock-control none --import-source on -k regex:k_bitmatrix_lists64 -s 2 -c 1 -o /tmp/prof_bm python scratch/quick_bm.py > gpurun_out/ncu_bm.log 2>&1
ncu -i /tmp/prof_bm.ncu-rep --page raw --csv > gpurun_out/bm_raw.csv 2>&1
ncu -i /tmp/prof_bm.ncu-rep --page source --csv --print-source sass > gpurun_out/bm_src.csv 2>&1
echo done
