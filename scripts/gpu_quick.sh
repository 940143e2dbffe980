# parity (no -x) + A/B timing on the two headline configs
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.txt 2>&1
timeout 900 python -m pytest tests -m gpu -q --timeout 300 > gpurun_out/pytest_gpu.txt 2>&1
tail -15 gpurun_out/pytest_gpu.txt
timeout 300 python scripts/exp_ab.py mha7b_b32 2>&1 | tail -3
timeout 300 python scripts/exp_ab.py mha7b_b16 2>&1 | tail -3
