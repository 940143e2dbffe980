mkdir -p gpurun_out/r03h
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
timeout -k 10 300 python scripts/timeline.py mha7b_b32 > gpurun_out/r03h/timeline.jsonl 2> gpurun_out/r03h/timeline.err
python -c "
import json
for l in open('gpurun_out/r03h/timeline.jsonl'):
    d=json.loads(l); print(d['config'], json.dumps(d.get('ramp_min_med_max')), json.dumps(d['phases_us_median']))
"
for c in mha7b_b32 mha7b_b16 mha7b_b32_fp8; do
  timeout -k 10 600 python scripts/ab.py $c 3 noearly -DBIFATTN_NO_EARLY_PLAN >> gpurun_out/r03h/ab.jsonl 2>> gpurun_out/r03h/ab.err
done
cat gpurun_out/r03h/ab.jsonl
