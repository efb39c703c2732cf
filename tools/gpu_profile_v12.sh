# Round-1 v12 profiles: launch list of a full bench run (main scan + f3/f4/f1 legs) and --set full
# captures of the main path's dominant kernel and of the f-row kernels, summarised ON THE BOX (the
# reports themselves exceed gpurun's 64 MiB return limit).
mkdir -p gpurun_out
CMD="python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-e2e --quiet"
$CMD > gpurun_out/plain.log 2>&1; echo plain_rc=$?
timeout 1200 ncu --metrics gpu__time_duration.sum --clock-control none -c 3000 --csv --log-file gpurun_out/launches_v12.csv $CMD > gpurun_out/ncu_launches.log 2>&1; echo ncu1_rc=$?
python tools/ncu_summary.py gpurun_out/launches_v12.csv gpurun_out/r01_v12 > /dev/null 2>&1
for k in ${KERNELS:-k_ladder k_relin3 k_rot1_ks k_exp_mask k_cmp_rot}; do
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:"^${k}" -s 1 -c 1 -o /tmp/prof_$k $CMD > gpurun_out/ncu_full_$k.log 2>&1; echo "$k rc=$?"
  python tools/ncu_summary.py /tmp/prof_$k.ncu-rep gpurun_out/r01_v12_$k > /dev/null 2>&1
  python tools/ncu_lines_stall.py /tmp/prof_$k.ncu-rep 25 > gpurun_out/r01_v12_${k}_lines.txt 2>&1
  rm -f /tmp/prof_$k.ncu-rep
done
