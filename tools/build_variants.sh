#!/bin/bash
# build A/B library variants here (CPU cross-compile): NAME=FLAGS pairs, e.g.
#   bash tools/build_variants.sh "nopshift=-DBM_NO_SHOUP_PSHIFT" "rb64=-DBM_RB64"
for spec in "$@"; do
  name=${spec%%=*}; flags=${spec#*=}
  BM_VARIANT=$name BM_NVCC_FLAGS="$flags" python -m paper_2408_06167_b200.build > /tmp/build_$name.log 2>&1 && echo "built $name" || { echo "FAILED $name"; tail -5 /tmp/build_$name.log; }
done
