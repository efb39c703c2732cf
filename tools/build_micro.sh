# build the diagnostic microbenchmarks (not the library)
set -e
NVCC=/usr/local/cuda/bin/nvcc
ARCH="-gencode arch=compute_100a,code=sm_100a"
for m in 1 2; do
$NVCC $ARCH -O3 -std=c++17 -DMINB3=$m -o tools/ntt_bench_m$m tools/ntt_bench.cu paper_2408_06167_b200/csrc/host.cpp -I include -lquadmath
done
$NVCC $ARCH -O3 -std=c++17 -o tools/pipe_bench tools/pipe_bench.cu
$NVCC $ARCH -O3 -std=c++17 -I include -o tools/modmul_bench tools/modmul_bench.cu
# diagnostic: the transform without its shared-memory exchanges (1: barriers kept, 2: nothing) -- wrong results,
# the compute-only ceiling of the core
for x in 1 2; do
$NVCC $ARCH -O3 -std=c++17 -DMINB3=1 -DBM_DIAG_XCHG=$x -o tools/ntt_bench_x$x tools/ntt_bench.cu paper_2408_06167_b200/csrc/host.cpp -I include -lquadmath
done
# diagnostic: twiddles without loads (3), and without loads or exchanges (4)
$NVCC $ARCH -O3 -std=c++17 -DMINB3=1 -DBM_DIAG_TW -o tools/ntt_bench_x3 tools/ntt_bench.cu paper_2408_06167_b200/csrc/host.cpp -I include -lquadmath
$NVCC $ARCH -O3 -std=c++17 -DMINB3=1 -DBM_DIAG_TW -DBM_DIAG_XCHG=2 -o tools/ntt_bench_x4 tools/ntt_bench.cu paper_2408_06167_b200/csrc/host.cpp -I include -lquadmath
