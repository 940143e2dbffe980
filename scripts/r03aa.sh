mkdir -p gpurun_out/r03aa
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
python scripts/host_overhead.py mha7b_b32 > gpurun_out/r03aa/host.jsonl 2>&1
python scripts/host_overhead.py mha7b_b16 >> gpurun_out/r03aa/host.jsonl 2>&1
cat gpurun_out/r03aa/host.jsonl
for c in mha7b_b32 mha7b_b16; do timeout -k 10 600 python scripts/ab.py $c 3 noncoop -DBIFATTN_NONCOOP >> gpurun_out/r03aa/ab.jsonl 2>> gpurun_out/r03aa/ab.err; done
python -c "
import json
for l in open('gpurun_out/r03aa/ab.jsonl'):
    d=json.loads(l); ks=[k for k in d if isinstance(d[k], dict)]; print(d['config'], [(k, round(d[k]['us_median'],2), round(d[k]['graph_median'],2)) for k in ks])"
