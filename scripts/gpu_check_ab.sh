# GPU check of a change: hang probe of PROBE_CFGS, pytest -m gpu, and interleaved A/Bs (scripts/ab.py) of AB_CFGS against AB_DEFS (-D flags or --lib PATH); results under gpurun_out/$TAG
set -x
OUT=gpurun_out/${TAG:-r03m}
mkdir -p $OUT
python -c "import __graft_entry__ as g; g.build()" > $OUT/build.txt 2>&1
for c in ${PROBE_CFGS:-mqa gqa}; do PROBE_STEPS=3 timeout -k 5 90 python scripts/hang_probe.py $c 20 >> $OUT/probe.txt 2>&1; echo "exit $?" >> $OUT/probe.txt; done
cut -c1-200 $OUT/probe.txt
grep -q '"finished": false' $OUT/probe.txt && exit 1
timeout -k 10 900 python -m pytest tests -m gpu -q -x --timeout 120 -rA > $OUT/pytest_gpu.txt 2>&1
tail -2 $OUT/pytest_gpu.txt; grep -E "FAILED|Error" $OUT/pytest_gpu.txt | head -5
for c in ${AB_CFGS:-mqa gqa long}; do
  timeout -k 10 900 python scripts/ab.py $c 3 ${AB_NAME:-noqtma} ${AB_DEFS:--DBIFATTN_NO_QTMA} >> $OUT/ab.jsonl 2>> $OUT/ab.err
done
python -c "
import json
for l in open('$OUT/ab.jsonl'):
    d=json.loads(l); ks=[k for k in d if isinstance(d[k], dict)]; print(d['config'], [(k, round(d[k]['us_median'],2)) for k in ks])"
