mkdir -p gpurun_out/r03g
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
timeout -k 10 300 python scripts/timeline.py mha7b_b32 > gpurun_out/r03g/timeline.jsonl 2> gpurun_out/r03g/timeline.err
python -c "
import json
for l in open('gpurun_out/r03g/timeline.jsonl'):
    d=json.loads(l); print(d['config'], json.dumps(d.get('ramp_min_med_max')))
"
