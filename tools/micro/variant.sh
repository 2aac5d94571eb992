set -x
cd $GRAFT_REPO_ROOT
K="python -m pytest tests/test_gpu_parity.py -q -p no:cacheprovider -k top_r_diagonal"
$K 2>&1 | tail -1
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -Xcompiler -fPIC -shared -DMEG_JACOBI_FP64 -o paper_2012_10469_b200/libmegb200.so paper_2012_10469_b200/csrc/megb200_kernels.cu paper_2012_10469_b200/csrc/megb200_coop.cu paper_2012_10469_b200/csrc/megb200_runtime.cu
$K 2>&1 | tail -1
