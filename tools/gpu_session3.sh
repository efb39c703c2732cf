#!/bin/bash
# full GPU suite on the product, the same suite on the debug build (bounds checks + barrier jitter),
# the headline bench and the configs[0] line
set -x
mkdir -p gpurun_out
python -m paper_2408_06167_b200.build > gpurun_out/build.log 2>&1
timeout 2400 python -m pytest tests -q -m gpu > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
BM_LIB_PATH=paper_2408_06167_b200/variants/libblindmatch_dbg.so timeout 3000 python -m pytest tests -q -m gpu -k "not full_grid" > gpurun_out/pytest_dbg.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_dbg.log
timeout 1500 python bench.py --steps 5 --warmup 3 > gpurun_out/bench.json 2> gpurun_out/bench.err; echo "bench rc=$?" >> gpurun_out/bench.err
timeout 600 python bench.py --config 1 --steps 5 --warmup 3 --no-extras > gpurun_out/c1.json 2> gpurun_out/c1.err; echo "rc=$?" >> gpurun_out/c1.err
