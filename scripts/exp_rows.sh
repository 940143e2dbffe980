mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.txt 2>&1
for c in gqa mqa long; do
  BIFATTN_CTX_ROWS=2 timeout 300 python bench.py --config $c --steps 10 --warmup 3 --no-e2e --no-cpu-baseline --no-replicated --soak 0 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$c', round(d['us_per_step'],1), d['kernels'])"
done
EXP_MC=16384 EXP_MD=0 BIFATTN_CTX_ROWS=2 EXP_CFG=gqa python scripts/exp_shapes.py 16384,0 | cut -c1-100
