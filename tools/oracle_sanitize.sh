#!/bin/bash
# The oracle's pins under AddressSanitizer + UndefinedBehaviorSanitizer (host-side):
# an instrumented liboracle_san.so, loaded into Python with the ASan runtime preloaded.
cd "$(dirname "$0")/.."
export ORACLE_SANITIZE=1
export ASAN_OPTIONS=detect_leaks=0:abort_on_error=1
export UBSAN_OPTIONS=halt_on_error=1:print_stacktrace=1
LD_PRELOAD="$(gcc -print-file-name=libasan.so) $(gcc -print-file-name=libubsan.so)" \
  python -m pytest tests/test_oracle_ring.py tests/test_oracle_prng.py tests/test_oracle_ckks.py \
  tests/test_oracle_expand.py tests/test_oracle_compress.py -q -x -p no:cacheprovider "$@"
