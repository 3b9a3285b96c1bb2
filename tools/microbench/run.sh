# build + run the INT / tensor-pipe microbenchmarks on the GPU box
cd $GRAFT_REPO_ROOT/tools/microbench
NV="nvcc -gencode arch=compute_100a,code=sm_100a -O3"
$NV -o int_peaks int_peaks.cu && timeout 120 ./int_peaks
$NV -o tc_i8 tc_i8.cu && timeout 120 ./tc_i8
