#!/bin/bash
# configs[3] (the metric's workload) under each evaluation order: the product (0), the paper order (1),
# and the f2 rotation sums (2 hoisted, 4 baby-step giant-step); verification on, no e2e / extras
mkdir -p gpurun_out
python -m paper_2408_06167_b200.build > gpurun_out/build.log 2>&1
OUT=gpurun_out/r02_c4_orders.jsonl; : > $OUT
for o in 2 4 0 1; do
  S=5; [ $o = 1 ] && S=3
  timeout 900 python bench.py --order $o --steps $S --warmup 3 --no-e2e --no-extras --no-cpu-baseline --no-single \
    >> $OUT 2>> gpurun_out/c4_orders.err; echo "order $o rc=$?" >> gpurun_out/c4_orders.err
done
