set -x
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.txt 2>&1
timeout 900 python -m pytest tests -m gpu -q -x --timeout 300 > gpurun_out/pytest_gpu.txt 2>&1
tail -5 gpurun_out/pytest_gpu.txt
timeout 300 python scripts/bench_multitoken.py > gpurun_out/mt.jsonl 2>&1; cat gpurun_out/mt.jsonl
MT_CFG=gqa timeout 300 python scripts/bench_multitoken.py >> gpurun_out/mt.jsonl 2>&1; tail -4 gpurun_out/mt.jsonl
