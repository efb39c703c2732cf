# build the NTT microbenchmark variants (diagnostic tools, not the library)
for m in 1 2; do
/usr/local/cuda/bin/nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -DMINB3=$m -o tools/ntt_bench_m$m tools/ntt_bench.cu paper_2408_06167_b200/csrc/host.cpp -I include -lquadmath
done
