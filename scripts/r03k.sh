set -x
OUT=gpurun_out/${TAG:-r03k}
mkdir -p $OUT
python -c "import __graft_entry__ as g; g.build()" > $OUT/build.txt 2>&1
for c in gqa mha7b_b32; do PROBE_STEPS=3 timeout -k 5 90 python scripts/hang_probe.py $c 20 >> $OUT/probe.txt 2>&1; echo "exit $?" >> $OUT/probe.txt; done
cut -c1-300 $OUT/probe.txt
grep -q '"finished": false' $OUT/probe.txt && exit 1
timeout -k 10 900 python -m pytest tests -m gpu -q -x --timeout 120 -rA > $OUT/pytest_gpu.txt 2>&1
tail -3 $OUT/pytest_gpu.txt; grep -E "FAILED|Error" $OUT/pytest_gpu.txt | head -5
for s in "4 32 8 1024 8192" "8 16 8 512 4096" "16 8 8 2048 2048" "8 32 16 1024 4096"; do
  timeout -k 10 600 python scripts/ab_custom.py $s 3 nodyn -DBIFATTN_NO_DYN >> $OUT/ab.jsonl 2>> $OUT/ab.err
done
cut -c1-260 $OUT/ab.jsonl
timeout -k 10 600 python bench.py --config gqa --no-e2e --no-replicated --no-cpu-baseline --no-stream-peak --no-others > $OUT/bench_gqa.json 2> $OUT/bench_gqa.err
python -c "
import json; d=json.load(open('$OUT/bench_gqa.json')); print(d['us_per_step'], json.dumps(d.get('kernels')))"
