# Final profiles of a round: the default bench line, the ncu launch list of the main scan (bench with the
# NEXT-row legs off, so the shares are the hot path's) and --set full summaries of the top kernels,
# summarised on the box.  TAG names the files (profiles/r01_<TAG>_*).
mkdir -p gpurun_out
TAG=${TAG:-v13}
timeout 900 python bench.py > gpurun_out/r01_bench_${TAG}.json 2> gpurun_out/bench_${TAG}.err; echo bench_rc=$?
CMD="python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-e2e --no-f3 --no-f1 --no-single --quiet"
$CMD > gpurun_out/plain.log 2>&1; echo plain_rc=$?
timeout 1200 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file /tmp/launches.csv $CMD > gpurun_out/ncu_launches.log 2>&1; echo ncu1_rc=$?
python tools/ncu_summary.py /tmp/launches.csv gpurun_out/r01_${TAG} > /dev/null 2>&1
cp /tmp/launches.csv gpurun_out/r01_${TAG}_launches.csv
for k in ${KERNELS:-k_ladder k_relin k_tensor k_digits}; do
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:"^${k}" -s 1 -c 1 -o /tmp/prof_$k $CMD > gpurun_out/ncu_full_$k.log 2>&1; echo "$k rc=$?"
  python tools/ncu_summary.py /tmp/prof_$k.ncu-rep gpurun_out/r01_${TAG}_$k > /dev/null 2>&1
  python tools/ncu_lines_stall.py /tmp/prof_$k.ncu-rep 25 > gpurun_out/r01_${TAG}_${k}_lines.txt 2>&1
  rm -f /tmp/prof_$k.ncu-rep
done
