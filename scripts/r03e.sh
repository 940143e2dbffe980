set -x
OUT=gpurun_out/${TAG:-r03e}
mkdir -p $OUT
python -c "import __graft_entry__ as g; g.build()" > $OUT/build.txt 2>&1
for c in mha7b_b32 mha7b_b16 long; do
  PROBE_STEPS=3 timeout -k 5 90 python scripts/hang_probe.py $c 20 >> $OUT/probe.txt 2>&1
  echo "exit $?" >> $OUT/probe.txt
done
cut -c1-400 $OUT/probe.txt
grep -q '"finished": false' $OUT/probe.txt && exit 1
timeout -k 10 900 python -m pytest tests -m gpu -q -x --timeout 120 -rA > $OUT/pytest_gpu.txt 2>&1
tail -3 $OUT/pytest_gpu.txt
timeout -k 10 300 python -c "import __graft_entry__ as g; g.smoke()" > $OUT/smoke.txt 2>&1
tail -5 $OUT/smoke.txt
timeout -k 10 300 python scripts/timeline.py mha7b_b32 mha7b_b16 > $OUT/timeline.jsonl 2> $OUT/timeline.err
python -c "
import json
for l in open('$OUT/timeline.jsonl'):
    d=json.loads(l); print(d['config'], json.dumps(d['dyn_min_med_max_n']), json.dumps(d['phases_us_median']), json.dumps(d['abs_us_min_med_max']), json.dumps(d.get('ramp_min_med_max')))
"
timeout -k 10 600 python bench.py > $OUT/bench.json 2> $OUT/bench.err
cut -c1-700 $OUT/bench.json
python -c "
import json; d=json.load(open('$OUT/bench.json'))
for k,v in d.get('other_configs',{}).items(): print(k, v.get('us_per_step'), v.get('graph_us_per_step'), v.get('plan','')[:60])
"
