# round-3 check of a change: build, GPU tests, smoke, A/B against a variant build, bench line
set -x
OUT=gpurun_out/${TAG:-r03}
mkdir -p $OUT
python -c "import __graft_entry__ as g; g.build()" > $OUT/build.txt 2>&1
timeout -k 10 600 python -m pytest tests -m gpu -q -x --timeout 120 -rA > $OUT/pytest_gpu.txt 2>&1
tail -3 $OUT/pytest_gpu.txt
timeout -k 10 300 python -c "import __graft_entry__ as g; g.smoke()" > $OUT/smoke.txt 2>&1
tail -5 $OUT/smoke.txt
for c in ${AB_CFGS:-mha7b_b32 mha7b_b16}; do
  timeout -k 10 900 python scripts/ab.py $c ${AB_ROUNDS:-3} ${AB_NAME:-nodyn} ${AB_DEFS:--DBIFATTN_NO_DYN} >> $OUT/ab.jsonl 2>> $OUT/ab.err
done
cat $OUT/ab.jsonl
timeout -k 10 900 python bench.py > $OUT/bench.json 2> $OUT/bench.err
cut -c1-600 $OUT/bench.json
