#!/bin/bash
# A/B: component 0 of the throughput ladder in two accumulators (product) vs the 6-transform step (nosplit)
mkdir -p gpurun_out
python -m paper_2408_06167_b200.build > gpurun_out/build.log 2>&1 || exit 1
timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_gpu_worstcase.py tests/test_gpu_configs.py -q -m gpu -x > gpurun_out/pytest_split.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_split.log
VARIANTS="base ladonly" ROUNDS=2 STEPS=5 BENCH_ARGS="--config 4" bash tools/ab.sh
