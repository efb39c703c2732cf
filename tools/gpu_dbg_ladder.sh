#!/bin/bash
# debug-build checks at the P-scaled ladder: (1) the failing f2 hoisted test under checks-only and jitter-only
# builds (which ingredient trips it), (2) the ladder / end-to-end / worst-case subset on the full debug build
mkdir -p gpurun_out
: > gpurun_out/pytest_dbg_ladder.log
for v in dbgchk dbgjit dbg; do
  echo "## $v: test_hoisted_rotation_order_parity" >> gpurun_out/pytest_dbg_ladder.log
  BM_LIB_PATH=paper_2408_06167_b200/variants/libblindmatch_$v.so timeout 600 python -m pytest tests/test_gpu_parity.py -q -m gpu -k "hoisted_rotation_order_parity" 2>&1 | tail -12 >> gpurun_out/pytest_dbg_ladder.log
done
echo "## dbg: ladder / end-to-end / worst-case subset (the product order)" >> gpurun_out/pytest_dbg_ladder.log
BM_LIB_PATH=paper_2408_06167_b200/variants/libblindmatch_dbg.so timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_worstcase.py -q -m gpu --durations=5 -k "(ladder or worst or end_to_end or tail or bench_config or layout or qm1 or alt) and not hoisted_rotation" >> gpurun_out/pytest_dbg_ladder.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_dbg_ladder.log
grep -E "^##|passed|failed|FAILED|rc=" gpurun_out/pytest_dbg_ladder.log
