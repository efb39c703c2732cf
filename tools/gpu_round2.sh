#!/bin/bash
# round-2 GPU session: microbenchmark, GPU tests, headline bench (logs under gpurun_out/)
set -x
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/smi.txt 2>&1
python -m paper_2408_06167_b200.build > gpurun_out/build.log 2>&1
timeout 120 tools/modmul_bench > gpurun_out/modmul_bench.txt 2>&1
timeout 1500 python -m pytest tests -x -q -m gpu ${PYTEST_ARGS} > gpurun_out/pytest_gpu.log 2>&1
echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
timeout 1200 python bench.py --steps ${STEPS:-3} --warmup ${WARMUP:-2} ${BENCH_ARGS} > gpurun_out/bench.json 2> gpurun_out/bench.err
echo "bench rc=$?" >> gpurun_out/bench.err
