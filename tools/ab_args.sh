#!/bin/bash
# A/B of bench arguments on the product library: ARGSETS="--chunk 296|--chunk 16384" (| separated)
mkdir -p gpurun_out
: > gpurun_out/ab_args.txt
IFS='|' read -ra SETS <<< "${ARGSETS}"
for r in $(seq ${ROUNDS:-2}); do
for i in "${!SETS[@]}"; do
  a=${SETS[$i]}
  timeout 900 python bench.py --steps ${STEPS:-10} --warmup 3 --no-verify --no-e2e --no-single --no-extras \
      --no-cpu-baseline $a > gpurun_out/ab_args_$i.json 2> gpurun_out/ab_args_$i.err
  python - "$i" "$a" >> gpurun_out/ab_args.txt <<'PY'
import json, sys
i, a = sys.argv[1], sys.argv[2]
try:
    d = json.loads(open(f"gpurun_out/ab_args_{i}.json").read().strip().splitlines()[-1])
    pc = d["roofline"]["per_class"]
    print(f"[{a:40s}] {d['ms_per_step']:10.3f} ms  {d['value']/1e6:8.2f} M  " +
          "  ".join(f"{k} {x['ms_per_step']:.3f}" for k, x in pc.items()))
except Exception as e:
    print(a, "FAILED", e)
PY
done
done
cat gpurun_out/ab_args.txt
