# quick parity + stage times, then ncu --set full (with source) of the given kernels in one C4 step
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
TAG=${1:-q}; RE=${2:-k_leaf_sort}; CNT=${3:-1}
bash tools/gpu/quick_c4.sh $TAG
bash tools/gpu/prof_r2.sh "$RE" ${TAG}_prof $CNT
