# ncu capture of selected kernels (KSEL regex) after a plain run of the same command
mkdir -p gpurun_out
CMD="python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-e2e --quiet ${BENCH_ARGS}"
$CMD > gpurun_out/plain.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"${KSEL:-k_ladder}" -s ${KSKIP:-6} -c ${KCOUNT:-1} -o gpurun_out/prof $CMD > gpurun_out/ncu_full.log 2>&1; echo ncu_rc=$?
