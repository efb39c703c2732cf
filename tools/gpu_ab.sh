# A/B of env variants on the bench: VARIANTS="BM_X=1 BM_X=2 ..." (each one bench run, no e2e/cpu baseline)
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1 || echo build_failed
for v in ${VARIANTS:-NONE=0}; do
  env $v timeout 600 python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-e2e ${BENCH_ARGS} > gpurun_out/ab.json 2>/dev/null
  python -c "
import json; d=json.load(open('gpurun_out/ab.json')); print('$v', d['value'], d['ms_per_step']); [print('   ', k, v) for k,v in d['roofline']['per_class'].items()]"
done
