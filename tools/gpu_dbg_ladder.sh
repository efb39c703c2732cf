#!/bin/bash
# the ladder / worst-case / end-to-end parity tests on the debug build (bounds checks + barrier jitter) at the
# P-scaled ladder: the subset of the -m gpu suite that exercises K3 -> k_ladder_t<false, true>
mkdir -p gpurun_out
BM_LIB_PATH=paper_2408_06167_b200/variants/libblindmatch_dbg.so timeout 1300 python -m pytest tests/test_gpu_parity.py tests/test_gpu_worstcase.py -q -m gpu -x --durations=8 -k "ladder or worst or end_to_end or tail or bench_config or hoisted or layout or qm1 or alt" > gpurun_out/pytest_dbg_ladder.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_dbg_ladder.log
tail -15 gpurun_out/pytest_dbg_ladder.log
