# GPU round: parity tests, full bench line, pipe/NTT microbenchmarks, ncu launch list + one
# --set full capture of the top kernel (TOPK).
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q -x > gpurun_out/gpu_tests.log 2>&1; echo tests_rc=$?; tail -3 gpurun_out/gpu_tests.log
timeout 900 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err; echo bench_rc=$?; tail -3 gpurun_out/bench.err; cat gpurun_out/bench.json
timeout 120 ./tools/pipe_bench > gpurun_out/pipe_bench.txt 2>&1
timeout 300 ./tools/ntt_bench_m1 2368 20 > gpurun_out/ntt_bench.txt 2>&1
CMD="python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-e2e --quiet"
$CMD > gpurun_out/plain.log 2>&1 && \
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 300 --csv --log-file gpurun_out/launches.csv $CMD > gpurun_out/ncu_launches.log 2>&1; echo ncu1_rc=$?
timeout 900 ncu --set full --clock-control none --import-source on -k regex:${TOPK:-k_ladder} -s 2 -c 1 -o gpurun_out/prof $CMD > gpurun_out/ncu_full.log 2>&1; echo ncu2_rc=$?
