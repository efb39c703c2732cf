# ncu --set full of the top kernel under several env variants: VARIANTS="A=1 A=2", KSEL regex
mkdir -p gpurun_out
CMD="python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-e2e --quiet ${BENCH_ARGS}"
i=0
for v in ${VARIANTS:-NONE=0}; do
  env $v $CMD > gpurun_out/plain_$i.log 2>&1 && \
  env $v timeout 900 ncu --set full --clock-control none --import-source on -k regex:"${KSEL:-k_ladder}" -s ${KSKIP:-3} -c 1 -o gpurun_out/prof_$i $CMD > gpurun_out/ncu_full_$i.log 2>&1; echo "$v ncu_rc=$?"
  i=$((i+1))
done
