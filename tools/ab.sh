#!/bin/bash
# A/B of library builds on the bench (tools/build_variants.sh builds them here; they travel in-tree):
#   VARIANTS="base v1 v2" ROUNDS=2 BENCH_ARGS="--config 2" bash tools/ab.sh
# base = the product library; other names = paper_2408_06167_b200/variants/libblindmatch_<name>.so
mkdir -p gpurun_out
: > gpurun_out/ab.txt
for r in $(seq ${ROUNDS:-2}); do
for v in ${VARIANTS:-base}; do
  if [ "$v" = base ]; then LP=""; else LP="paper_2408_06167_b200/variants/libblindmatch_$v.so"; fi
  BM_LIB_PATH=$LP timeout 900 python bench.py --steps ${STEPS:-10} --warmup 3 --no-verify --no-e2e --no-single \
      --no-extras --no-cpu-baseline ${BENCH_ARGS:---config 2} > gpurun_out/ab_$v.json 2> gpurun_out/ab_$v.err
  python - "$v" >> gpurun_out/ab.txt <<'PY'
import json, sys
v = sys.argv[1]
try:
    d = json.loads(open(f"gpurun_out/ab_{v}.json").read().strip().splitlines()[-1])
    pc = d["roofline"]["per_class"]
    print(f"{v:12s} {d['ms_per_step']:10.3f} ms  {d['value']/1e6:8.2f} M  frac {d['roofline']['frac']:.4f}  " +
          "  ".join(f"{k} {x['ms_per_step']:.3f}" for k, x in pc.items()))
except Exception as e:
    print(v, "FAILED", e)
PY
done
done
cat gpurun_out/ab.txt
