mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.txt 2>&1
timeout 200 python -m pytest tests/test_gpu_parity.py -q -x -k "rows130 and rows" --timeout 60 > gpurun_out/pytest_rows.txt 2>&1
tail -4 gpurun_out/pytest_rows.txt | cut -c1-300
timeout 300 python -m pytest tests/test_gpu_parity.py tests/test_gpu_multitoken.py -q -x --timeout 60 > gpurun_out/pytest_rows2.txt 2>&1
tail -2 gpurun_out/pytest_rows2.txt | cut -c1-300
for c in mqa gqa long; do echo "$c $(EXP_CFG=$c timeout 120 python scripts/exp_shapes.py 0,0 | cut -c1-100)"; done
