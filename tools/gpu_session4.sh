#!/bin/bash
set -x
mkdir -p gpurun_out
python -m paper_2408_06167_b200.build > gpurun_out/build.log 2>&1
VARIANTS="base canons" ROUNDS=3 STEPS=20 BENCH_ARGS="--config 2" bash tools/ab.sh
timeout 2400 python -m pytest tests -q -m gpu > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
BL="--steps 1 --warmup 1 --no-verify --no-e2e --no-single --no-extras --no-cpu-baseline"
for k in k_tensor k_digits; do
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:$k -c 1 -f -o gpurun_out/ncu_$k python bench.py $BL > gpurun_out/ncu_$k.log 2>&1
done
