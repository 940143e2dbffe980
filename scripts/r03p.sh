set -x
OUT=gpurun_out/r03p
mkdir -p $OUT
python -c "import __graft_entry__ as g; g.build()" > $OUT/build.txt 2>&1
timeout -k 10 900 python -m pytest tests -m gpu -q -x --timeout 120 -rA > $OUT/pytest_gpu.txt 2>&1
tail -2 $OUT/pytest_gpu.txt; grep -E "FAILED|Error" $OUT/pytest_gpu.txt | head -5
grep -E "mqa: all|gqa: all" $OUT/pytest_gpu.txt | head
for c in mqa gqa; do
  timeout -k 10 900 python scripts/ab.py $c 3 poly0 -DCTXR_POLY=0 >> $OUT/ab.jsonl 2>> $OUT/ab.err
  timeout -k 10 900 python scripts/ab.py $c 3 poly5 -DCTXR_POLY=5 >> $OUT/ab.jsonl 2>> $OUT/ab.err
done
python -c "
import json
for l in open('$OUT/ab.jsonl'):
    d=json.loads(l); ks=[k for k in d if isinstance(d[k], dict)]; print(d['config'], [(k, round(d[k]['us_median'],2)) for k in ks])"
