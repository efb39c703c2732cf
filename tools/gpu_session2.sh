#!/bin/bash
# round-2 session: microbenchmarks of the paired transforms, the configs[0] hang, pair-kernel tests + A/B
set -x
mkdir -p gpurun_out
python -m paper_2408_06167_b200.build > gpurun_out/build.log 2>&1
/usr/local/cuda/bin/nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -DMINB3=1 -o tools/ntt_bench_m1 tools/ntt_bench.cu paper_2408_06167_b200/csrc/host.cpp -I include -lquadmath > gpurun_out/ntt_build.log 2>&1
timeout 300 tools/ntt_bench_m1 2368 20 > gpurun_out/ntt_bench.txt 2>&1
BM_BENCH_WATCHDOG=120 timeout 300 python bench.py --config 1 --steps 2 --warmup 1 > gpurun_out/c1.json 2> gpurun_out/c1.err
timeout 900 python -m pytest tests -q -m gpu -k "pair_kernels or config1 or decrypt_dev" > gpurun_out/pytest_pair.log 2>&1
VARIANTS="base acc29" ROUNDS=2 STEPS=20 BENCH_ARGS="--config 2" bash tools/ab.sh
ARGSETS="--config 2|--config 2 --opt pair_kernels=1" ROUNDS=2 STEPS=20 bash tools/ab_args.sh
