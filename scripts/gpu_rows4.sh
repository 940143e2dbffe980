mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.txt 2>&1
timeout 150 python -m pytest tests/test_gpu_parity.py tests/test_gpu_multitoken.py -q -x --timeout 30 > gpurun_out/pytest_rows2.txt 2>&1
tail -3 gpurun_out/pytest_rows2.txt | cut -c1-300
for c in mqa gqa long; do echo "$c $(EXP_CFG=$c timeout 40 python scripts/exp_shapes.py 0,0 | cut -c1-100)"; done
