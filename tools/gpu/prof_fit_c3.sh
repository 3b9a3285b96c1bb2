# ncu --set full (with source) of one mid-run k_group_fit launch of config 3
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
NAME=${1:-fitc3}
cat > /tmp/c3_once.py <<'P'
import sys, torch
sys.path.insert(0, '.')
import paper_2605_25974_b200 as pl
from paper_2605_25974_b200 import rng
x, z, f, c = rng.config_columns(3)
S = pl.PauliSumSoA.from_columns(100, x, z, f, c, device=torch.device('cuda', 0))
g, ng, pc = pl.group_assignment(S); torch.cuda.synchronize(); print(int(ng.item()))
P
timeout 900 ncu -f --set full --clock-control none --import-source on -k regex:k_group_fit --launch-skip 140 -c 1 -o /tmp/$NAME python /tmp/c3_once.py > gpurun_out/${NAME}_ncu.log 2>&1; echo "ncu rc=$?"
ncu -i /tmp/$NAME.ncu-rep --page raw --csv > gpurun_out/${NAME}_raw.csv 2>&1
ncu -i /tmp/$NAME.ncu-rep --page source --csv --print-source cuda,sass > gpurun_out/${NAME}_src.csv 2>&1
ls -la gpurun_out/${NAME}* | awk '{print $5, $9}'
