#!/bin/bash
# GPU session driver: STAGES (space-separated) of build pytest sanitize bench ncu_launch ncu_full
# logs under gpurun_out/ (merged back by gpurun)
set -x
mkdir -p gpurun_out
STAGES=${STAGES:-"build pytest bench"}
BARGS_LIGHT="--steps 1 --warmup 1 --no-verify --no-e2e --no-single --no-extras --no-cpu-baseline ${BENCH_ARGS}"
for st in $STAGES; do
case $st in
build) python -m paper_2408_06167_b200.build > gpurun_out/build.log 2>&1 ;;
micro) bash tools/build_micro.sh > gpurun_out/micro_build.log 2>&1; timeout 120 tools/modmul_bench > gpurun_out/modmul_bench.txt 2>&1 ;;
pytest) timeout ${PYTEST_TIMEOUT:-2400} python -m pytest tests -q -m gpu ${PYTEST_K:+-k "$PYTEST_K"} ${PYTEST_ARGS} > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log ;;
sanitize)
  timeout 1200 compute-sanitizer --tool memcheck --print-limit 20 python tools/sanitize.py all > gpurun_out/san_memcheck.log 2>&1; echo "rc=$?" >> gpurun_out/san_memcheck.log
  timeout 1200 compute-sanitizer --tool racecheck --racecheck-report all --print-limit 20 python tools/sanitize.py small > gpurun_out/san_racecheck.log 2>&1; echo "rc=$?" >> gpurun_out/san_racecheck.log
  timeout 900 compute-sanitizer --tool synccheck --print-limit 20 python tools/sanitize.py small > gpurun_out/san_synccheck.log 2>&1; echo "rc=$?" >> gpurun_out/san_synccheck.log ;;
bench) timeout 1500 python bench.py --steps ${STEPS:-3} --warmup ${WARMUP:-2} ${BENCH_ARGS} > gpurun_out/bench.json 2> gpurun_out/bench.err; echo "bench rc=$?" >> gpurun_out/bench.err ;;
ncu_launch) timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c ${NCU_COUNT:-300} --csv --log-file gpurun_out/ncu_launches.csv python bench.py $BARGS_LIGHT > gpurun_out/ncu_launch.log 2>&1 ;;
ncu_full)
  for k in ${NCU_KERNELS:-k_ladder_t k_relin}; do
    timeout 900 ncu --set full --clock-control none --import-source on -k regex:$k -c 1 -f -o gpurun_out/ncu_$k python bench.py $BARGS_LIGHT > gpurun_out/ncu_$k.log 2>&1
  done ;;
esac
done
