# build the diagnostic microbenchmarks (not the library)
set -e
NVCC=/usr/local/cuda/bin/nvcc
ARCH="-gencode arch=compute_100a,code=sm_100a"
for m in 1 2; do
$NVCC $ARCH -O3 -std=c++17 -DMINB3=$m -o tools/ntt_bench_m$m tools/ntt_bench.cu paper_2408_06167_b200/csrc/host.cpp -I include -lquadmath
done
$NVCC $ARCH -O3 -std=c++17 -o tools/pipe_bench tools/pipe_bench.cu
$NVCC $ARCH -O3 -std=c++17 -I include -o tools/modmul_bench tools/modmul_bench.cu
