#!/bin/bash
# A/B of the P-scaled throughput ladder (LADDER_PSCALE): parity first (the ladder / configs / worst-case
# tests on the product build), then base vs nops (= -DBM_LADDER_NO_PSCALE) on configs[1] and configs[3]
mkdir -p gpurun_out
timeout 1500 python -m pytest tests/test_gpu_parity.py tests/test_gpu_worstcase.py tests/test_gpu_configs.py -q -m gpu -x > gpurun_out/pscale_pytest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pscale_pytest.log
tail -3 gpurun_out/pscale_pytest.log
VARIANTS="base nops" ROUNDS=2 STEPS=10 BENCH_ARGS="--config 2" bash tools/ab.sh; cp gpurun_out/ab.txt gpurun_out/ab_pscale_c2.txt
VARIANTS="base nops" ROUNDS=2 STEPS=3 BENCH_ARGS="--config 4" bash tools/ab.sh; cp gpurun_out/ab.txt gpurun_out/ab_pscale_c4.txt
