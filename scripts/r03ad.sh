mkdir -p gpurun_out/r03ad
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
for c in mha7b_b32 mha7b_b16 mha7b_b32_fp8; do timeout -k 10 600 python scripts/ab.py $c 3 units12 --lib paper_2403_08845_b200/libbifattn_units12.so >> gpurun_out/r03ad/ab.jsonl 2>> gpurun_out/r03ad/ab.err; done
python -c "
import json
for l in open('gpurun_out/r03ad/ab.jsonl'):
    d=json.loads(l); ks=[k for k in d if isinstance(d[k], dict)]; print(d['config'], [(k, round(d[k]['us_median'],2), round(d[k]['graph_median'],2)) for k in ks])"
