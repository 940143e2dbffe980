mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.txt 2>&1
timeout 300 python -m pytest tests/test_gpu_parity.py tests/test_gpu_multitoken.py -q -x -k "rows or mqa" --timeout 60 > gpurun_out/pytest_rows.txt 2>&1
tail -3 gpurun_out/pytest_rows.txt
for c in mqa long; do
  timeout 300 python bench.py --config $c --steps 10 --warmup 3 --no-e2e --no-cpu-baseline --no-replicated --soak 0 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$c', round(d['us_per_step'],1), d['kernels'])"
done
BIFATTN_CTX_ROWS=2 EXP_CFG=gqa timeout 120 python scripts/exp_shapes.py 16384,0 16384,512 | cut -c1-100
