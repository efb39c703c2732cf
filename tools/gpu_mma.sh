#!/bin/bash
# tensor-core K1: its parity tests, then the bench with tensor_mma on / off
mkdir -p gpurun_out
python -m paper_2408_06167_b200.build > gpurun_out/build.log 2>&1 || exit 1
timeout 900 python -m pytest tests/test_gpu_tensor_mma.py -q -x > gpurun_out/pytest_mma.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_mma.log
: > gpurun_out/ab.txt
for v in 1 0; do  # tensor_mma on / off (DB registered either way)
  timeout 600 python bench.py --steps 5 --warmup 3 --no-verify --no-e2e --no-single --no-extras --no-cpu-baseline \
     --opt tensor_mma=$v > gpurun_out/ab_mma$v.json 2> gpurun_out/ab_mma$v.err
  python - "$v" >> gpurun_out/ab.txt <<'PY'
import json, sys
v = sys.argv[1]
try:
    d = json.loads(open(f"gpurun_out/ab_mma{v}.json").read().strip().splitlines()[-1])
    pc = d["roofline"]["per_class"]
    print(f"mma={v} {d['ms_per_step']:10.3f} ms  {d['value']/1e6:8.2f} M  " + "  ".join(f"{k} {x['ms_per_step']:.3f}" for k, x in pc.items()))
except Exception as e:
    print(v, "FAILED", e)
PY
done
cat gpurun_out/ab.txt
