# ncu launch list of the whole default bench step INCLUDING the NEXT-row legs (f3 expansion, f4
# enrollment, f1 compressed scan), so each f-row's kernels get their device-time breakdown.
# TAG names the files (profiles/r01_<TAG>_frows_*).
mkdir -p gpurun_out
TAG=${TAG:-v16}
CMD="python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-e2e --quiet"
$CMD > gpurun_out/frows_plain.json 2> gpurun_out/frows_plain.err; echo plain_rc=$?
timeout 1800 ncu --metrics gpu__time_duration.sum --clock-control none -c 20000 --csv --log-file /tmp/launches_f.csv $CMD > gpurun_out/ncu_frows.log 2>&1; echo ncu_rc=$?
python tools/ncu_summary.py /tmp/launches_f.csv gpurun_out/r01_${TAG}_frows > /dev/null 2>&1
gzip -c /tmp/launches_f.csv > gpurun_out/r01_${TAG}_frows_launches.csv.gz
