#!/bin/bash
# final evidence session: GPU suite, smoke, headline bench, launch list, configs sweep
set -x
mkdir -p gpurun_out
python -m paper_2408_06167_b200.build > gpurun_out/build.log 2>&1
timeout 2400 python -m pytest tests -q -m gpu > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/smoke.log
timeout 1500 python bench.py --steps 20 --warmup 5 > gpurun_out/bench.json 2> gpurun_out/bench.err; echo "bench rc=$?" >> gpurun_out/bench.err
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 300 --csv --log-file gpurun_out/ncu_launches.csv python bench.py --steps 1 --warmup 1 --no-verify --no-e2e --no-single --no-extras --no-cpu-baseline > gpurun_out/ncu_launch.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_ladder_t -c 1 -f -o gpurun_out/ncu_k_ladder_t python bench.py --steps 1 --warmup 1 --no-verify --no-e2e --no-single --no-extras --no-cpu-baseline > gpurun_out/ncu_l.log 2>&1
bash tools/gpu_configs.sh
