# quick GPU iteration: parity tests + bench (no cpu baseline) + optional A/B env + optional microbench
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q -x > gpurun_out/gpu_tests.log 2>&1; echo tests_rc=$?; tail -3 gpurun_out/gpu_tests.log
timeout 600 python bench.py --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/bench.json 2> gpurun_out/bench.err; echo bench_rc=$?; tail -2 gpurun_out/bench.err
python - <<'PY'
import json; d=json.load(open('gpurun_out/bench.json')); print(d['value'], d['ms_per_step'], d['roofline']['frac'], d['e2e'] and d['e2e']['ms_per_step'])
for k,v in d['roofline']['per_class'].items(): print(k, v)
PY
if [ -n "$AB" ]; then env $AB timeout 600 python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/bench_ab.json 2>/dev/null; python -c "
import json; d=json.load(open('gpurun_out/bench_ab.json')); print('AB', d['value'], d['ms_per_step']); [print(k, v) for k,v in d['roofline']['per_class'].items()]"; fi
for b in $MICRO; do echo "== $b"; timeout 120 $b 2368 20 2>&1 | tail -4; done
