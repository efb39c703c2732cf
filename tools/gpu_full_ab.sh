#!/bin/bash
# full GPU suite, then the A/B bench lines (VARIANTS, tools/ab.sh) and an ncu capture of $KN
mkdir -p gpurun_out
python -m paper_2408_06167_b200.build > gpurun_out/build.log 2>&1 || exit 1
timeout 2400 python -m pytest tests -q -m gpu -x > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
VARIANTS="${VARIANTS:-base}" ROUNDS=1 STEPS=5 BENCH_ARGS="--config 4" bash tools/ab.sh
[ -n "$KN" ] && KN=$KN TAG=${TAG:-x} bash tools/gpu_ncu_one.sh
exit 0
