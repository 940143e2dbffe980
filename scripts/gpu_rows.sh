mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.txt 2>&1
timeout 240 python -m pytest tests/test_gpu_parity.py -q -x -k "rows or mqa_small" --timeout 60 > gpurun_out/pytest_rows.txt 2>&1
tail -15 gpurun_out/pytest_rows.txt
