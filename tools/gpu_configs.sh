#!/bin/bash
# BASELINE.json configs[0..4] bench lines (p sweeps) -> gpurun_out/configs.jsonl
mkdir -p gpurun_out
: > gpurun_out/configs.jsonl
run() {  # label, args
  timeout ${TMO:-1500} python bench.py --no-extras "${@:2}" > gpurun_out/cfg_$1.json 2> gpurun_out/cfg_$1.err
  echo "rc=$?" >> gpurun_out/cfg_$1.err
  tail -1 gpurun_out/cfg_$1.json >> gpurun_out/configs.jsonl
}
SPECS=${SPECS:-"1:1 2:1 2:2 2:4 2:8 3:1 3:2 3:4 5:16 5:8 5:4"}
for spec in $SPECS; do
  c=${spec%%:*}; p=${spec#*:}
  case $c in
    5) run c${c}p$p --config $c --p $p --steps 2 --warmup 1 --no-e2e ;;
    *) run c${c}p$p --config $c --p $p --steps 5 --warmup 3 ;;
  esac
done
