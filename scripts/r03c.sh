# round-3: GPU tests, smoke, sanitizers of the changed plans, timeline, bench line
set -x
OUT=gpurun_out/${TAG:-r03c}
mkdir -p $OUT
python -c "import __graft_entry__ as g; g.build()" > $OUT/build.txt 2>&1
timeout -k 10 600 python -m pytest tests -m gpu -q -x --timeout 120 -rA > $OUT/pytest_gpu.txt 2>&1
tail -3 $OUT/pytest_gpu.txt
timeout -k 10 300 python -c "import __graft_entry__ as g; g.smoke()" > $OUT/smoke.txt 2>&1
tail -5 $OUT/smoke.txt
for tool in memcheck racecheck synccheck; do
  timeout -k 10 600 compute-sanitizer --tool $tool --print-limit 20 python scripts/sanitize_cases.py ${SAN_CASES:-fused_dyn rows_dec_tc fused_tc multitoken} > $OUT/sanitizer_$tool.txt 2>&1
  echo "exit $?" >> $OUT/sanitizer_$tool.txt
  tail -3 $OUT/sanitizer_$tool.txt
done
timeout -k 10 600 python scripts/timeline.py mha7b_b32 mha7b_b16 > $OUT/timeline.jsonl 2> $OUT/timeline.err
python -c "
import json
for l in open('$OUT/timeline.jsonl'):
    d=json.loads(l); print(d['config'], json.dumps(d['dyn_min_med_max_n']), json.dumps(d['phases_us_median']), json.dumps(d['abs_us_min_med_max']), json.dumps(d.get('ramp_min_med_max')))
"
timeout -k 10 900 python bench.py > $OUT/bench.json 2> $OUT/bench.err
cut -c1-700 $OUT/bench.json
python -c "
import json; d=json.load(open('$OUT/bench.json'))
for k,v in d.get('other_configs',{}).items(): print(k, v.get('us_per_step'), v.get('graph_us_per_step'), v.get('plan','')[:60])
"
