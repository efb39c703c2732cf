#!/bin/bash
# one ncu --set full capture of kernel $KN in a light bench run, summarised on the box (TAG names the files)
mkdir -p gpurun_out
python -m paper_2408_06167_b200.build > gpurun_out/build.log 2>&1 || exit 1
CMD="python bench.py --steps 1 --warmup 1 --no-verify --no-e2e --no-single --no-extras --no-cpu-baseline ${BENCH_ARGS}"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"${KN}" -s ${SKIP:-2} -c 1 -f -o /tmp/prof $CMD > gpurun_out/ncu_${TAG}.log 2>&1; echo "ncu rc=$?"
python tools/ncu_summary.py /tmp/prof.ncu-rep gpurun_out/${TAG} > /dev/null 2>&1
python tools/ncu_lines_stall.py /tmp/prof.ncu-rep 30 > gpurun_out/${TAG}_lines.txt 2>&1
