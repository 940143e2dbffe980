set -x
OUT=gpurun_out/${TAG:-r03l}
mkdir -p $OUT
python -c "import __graft_entry__ as g; g.build()" > $OUT/build.txt 2>&1
timeout -k 10 900 python -m pytest tests -m gpu -q -x --timeout 120 -rA > $OUT/pytest_gpu.txt 2>&1
tail -3 $OUT/pytest_gpu.txt; grep -E "FAILED|Error" $OUT/pytest_gpu.txt | head -5
timeout -k 10 600 python bench.py > $OUT/bench.json 2> $OUT/bench.err
cut -c1-300 $OUT/bench.json
python -c "
import json; d=json.load(open('$OUT/bench.json'))
for k,v in d.get('other_configs',{}).items(): print(k, v.get('us_per_step'), v.get('graph_us_per_step'), json.dumps(v.get('kernels')), v.get('plan','')[:90])
"
