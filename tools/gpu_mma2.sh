#!/bin/bash
mkdir -p gpurun_out
python -m paper_2408_06167_b200.build > gpurun_out/build.log 2>&1 || exit 1
timeout 900 python -m pytest tests/test_gpu_tensor_mma.py -q -x > gpurun_out/pytest_mma.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_mma.log
VARIANTS="${VARIANTS:-base nohint}" ROUNDS=1 STEPS=5 BENCH_ARGS="--config 4" bash tools/ab.sh
KN=k_tensor_mma TAG=${TAG:-mma_v5} bash tools/gpu_ncu_one.sh
