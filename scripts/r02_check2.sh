# round-2 GPU check 2: build, GPU tests, the new bench line
set -x
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.txt 2>&1
timeout 1500 python -m pytest tests -m gpu -q -x --timeout 600 -rA > gpurun_out/pytest_gpu.txt 2>&1
grep -E "rows: max_abs|plan-covering|b32-n4" gpurun_out/pytest_gpu.txt > gpurun_out/parity_full.txt
timeout 900 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err
