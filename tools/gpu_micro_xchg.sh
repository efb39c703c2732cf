#!/bin/bash
# transform-core ceilings (diagnostic builds, wrong results by design): without the shared-memory exchanges,
# without the twiddle loads, without both
mkdir -p gpurun_out
OUT=gpurun_out/r02_ntt_bench_diag.txt
echo "# product core (MINB3=1)" > $OUT; ./tools/ntt_bench_m1 >> $OUT 2>&1
echo "# BM_DIAG_XCHG=1: barriers kept, no exchange data" >> $OUT; ./tools/ntt_bench_x1 >> $OUT 2>&1
echo "# BM_DIAG_XCHG=2: no exchange at all" >> $OUT; ./tools/ntt_bench_x2 >> $OUT 2>&1
echo "# BM_DIAG_TW: twiddles as constant-bank operands (no loads)" >> $OUT; ./tools/ntt_bench_x3 >> $OUT 2>&1
echo "# BM_DIAG_TW + BM_DIAG_XCHG=2: no twiddle loads, no exchanges" >> $OUT; ./tools/ntt_bench_x4 >> $OUT 2>&1
