# configs[1] layout sweep (d = 128, p in {1, 2, 4, 8}) for both op orders and
# f2's hoisted rotations: one bench line per point (device time, no e2e / NEXT legs), summarised.
mkdir -p gpurun_out
TAG=${TAG:-v17}
out=gpurun_out/r01_psweep_${TAG}.txt
echo "# configs[1] p sweep (bench.py --p P --order O --steps 5 --warmup 3): ms/step, templates*queries/s, ladder-or-hrot ms, single-query ms" > $out
for order in 0 1 2; do
  for p in 1 2 4 8; do
    timeout 600 python bench.py --p $p --order $order --steps 5 --warmup 3 --no-cpu-baseline --no-e2e --no-f3 --no-f1 > gpurun_out/ps.json 2>/dev/null || { echo "p=$p order=$order failed" >> $out; continue; }
    python - "$p" "$order" >> $out <<'PY'
import json, sys
d = json.load(open("gpurun_out/ps.json"))
pc = d["roofline"]["per_class"]
rot = pc.get("ladder", pc.get("hrot", {})).get("ms_per_step", 0.0)
print(f"p={sys.argv[1]:>2} order={['hoisted','paper','hoisted-rot(f2)'][int(sys.argv[2])]:16s} {d['ms_per_step']:9.3f} ms "
      f"{d['value']/1e6:8.2f} M/s  rot {rot:7.3f} ms  frac {d['roofline']['frac']:.3f} ({d['roofline']['kernel']})  "
      f"single {d['single_query']['ms']:.3f} ms")
PY
  done
done
cat $out
