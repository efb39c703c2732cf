#!/bin/bash
# round-2 re-entry check at HEAD: GPU suite, smoke, a short configs[3] bench line
mkdir -p gpurun_out
python -m paper_2408_06167_b200.build > gpurun_out/build.log 2>&1
timeout 2400 python -m pytest tests -q -m gpu -x > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/smoke.log
timeout 1500 python bench.py --steps 5 --warmup 3 > gpurun_out/head_bench.json 2> gpurun_out/head_bench.err; echo "bench rc=$?" >> gpurun_out/head_bench.err
