set -x
mkdir -p gpurun_out/r03b
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/r03b/build.txt 2>&1
timeout -k 10 300 python -m pytest tests/test_gpu_parity.py -q -x --timeout 120 -k "long" > gpurun_out/r03b/pytest_long.txt 2>&1; tail -3 gpurun_out/r03b/pytest_long.txt
timeout -k 10 600 python scripts/timeline.py mha7b_b32 mha7b_b16 > gpurun_out/r03b/timeline.jsonl 2> gpurun_out/r03b/timeline.err
python -c "
import json
for l in open('gpurun_out/r03b/timeline.jsonl'):
    d=json.loads(l); print(d['config'], json.dumps(d['dyn_min_med_max_n']), json.dumps(d['phases_us_median']), json.dumps(d['abs_us_min_med_max']))
"
