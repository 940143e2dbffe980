mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.txt 2>&1
timeout 900 python -m pytest tests -m gpu -q -x --timeout 300 > gpurun_out/pytest_gpu.txt 2>&1
tail -15 gpurun_out/pytest_gpu.txt
for cfg in mha7b_b16 mha7b_b32; do EXP_CFG=$cfg python scripts/exp_shapes.py 0,0 | cut -c1-80; done
