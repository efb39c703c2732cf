mkdir -p gpurun_out
./tools/ntt_bench_m1 2368 20 2>&1 | grep v3 > gpurun_out/ntt_m1.txt; cat gpurun_out/ntt_m1.txt
./tools/ntt_bench_m2 2368 20 2>&1 | grep v3 > gpurun_out/ntt_m2.txt; cat gpurun_out/ntt_m2.txt
CMD="python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-e2e --quiet"
$CMD > gpurun_out/plain.log 2>&1 && \
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches.csv $CMD > gpurun_out/ncu_launches.log 2>&1; echo ncu1_rc=$?
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_ladder|k_tensor_intt" -s 6 -c 2 -o gpurun_out/prof $CMD > gpurun_out/ncu_full.log 2>&1; echo ncu2_rc=$?
