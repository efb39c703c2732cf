#!/bin/bash
# f2 rotation-variant session: parity tests, then configs[1] p = 8 (s = 16) with the ladder, the
# hoisted sum and the baby-step giant-step sum (device time, verification on)
mkdir -p gpurun_out
python -m paper_2408_06167_b200.build > gpurun_out/build.log 2>&1
timeout 1500 python -m pytest tests -q -m gpu -k "${PYTEST_K:-hoisted_rotation or rows_fused}" > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
for o in ${ORDERS:-0 2 4}; do
  timeout 900 python bench.py --config 2 --order $o --steps 5 --warmup 3 --no-extras --no-cpu-baseline --no-e2e ${BENCH_ARGS} > gpurun_out/bench_o$o.json 2> gpurun_out/bench_o$o.err; echo "rc=$?" >> gpurun_out/bench_o$o.err
done
