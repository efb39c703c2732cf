#!/bin/bash
# last evidence of round 2 (after the P-scaled ladder and the two-count roofline): the default bench
# line as the driver runs it (20 steps, 5 warm-ups), the reference arm, and the GPU suite on the debug
# build (bounds checks + barrier jitter)
mkdir -p gpurun_out
TAG=${TAG:-c4_v6}
python -m paper_2408_06167_b200.build > gpurun_out/build.log 2>&1
timeout 1500 python bench.py --gpus 1 --steps 20 --warmup 5 > gpurun_out/r02_bench_${TAG}.json 2> gpurun_out/bench.err; echo "bench rc=$?" >> gpurun_out/bench.err
BM_LIB_PATH=paper_2408_06167_b200/variants/libblindmatch_dbg.so timeout 3000 python -m pytest tests -q -m gpu -k "not full_grid" > gpurun_out/pytest_dbg.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_dbg.log
tail -3 gpurun_out/pytest_dbg.log
