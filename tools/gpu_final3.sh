#!/bin/bash
# round-2 final evidence: GPU suite, smoke, the default bench line (20 steps), the reference arm, the ncu
# launch list of the configs[3] step and --set full summaries of its kernels (files gpurun_out/r02_${TAG}_*)
mkdir -p gpurun_out
TAG=${TAG:-c4_v5}
python -m paper_2408_06167_b200.build > gpurun_out/build.log 2>&1
timeout 2400 python -m pytest tests -q -m gpu > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/smoke.log
timeout 1500 python bench.py --steps 20 --warmup 5 > gpurun_out/r02_bench_${TAG}.json 2> gpurun_out/bench.err; echo "bench rc=$?" >> gpurun_out/bench.err
timeout 1200 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/r02_reference_arm_${TAG}.json 2> gpurun_out/ref.err; echo "ref rc=$?" >> gpurun_out/ref.err
CMD="python bench.py --steps 1 --warmup 1 --no-verify --no-e2e --no-single --no-extras --no-cpu-baseline --quiet"
timeout 1200 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file /tmp/launches.csv $CMD > gpurun_out/ncu_launches.log 2>&1; echo ncu1_rc=$?
python tools/ncu_summary.py /tmp/launches.csv gpurun_out/r02_${TAG} > /dev/null 2>&1
cp /tmp/launches.csv gpurun_out/r02_${TAG}_launches.csv
for k in ${KERNELS:-k_ladder_t k_relin k_tensor_mma k_digits}; do
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:"^${k}" -s 2 -c 1 -f -o /tmp/prof_$k $CMD > gpurun_out/ncu_full_$k.log 2>&1; echo "$k rc=$?"
  python tools/ncu_summary.py /tmp/prof_$k.ncu-rep gpurun_out/r02_${TAG}_$k > /dev/null 2>&1
  python tools/ncu_lines_stall.py /tmp/prof_$k.ncu-rep 25 > gpurun_out/r02_${TAG}_${k}_lines.txt 2>&1
  rm -f /tmp/prof_$k.ncu-rep
done
