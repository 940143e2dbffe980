# round-2: FP8 KV GPU parity + a quick timing of the FP8 C2b step
set -x
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.txt 2>&1
timeout 900 python -m pytest tests/test_gpu_kv8.py -q -x --timeout 300 -rA > gpurun_out/pytest_kv8.txt 2>&1
timeout 300 python bench.py --config mha7b_b32_fp8 --steps 30 --no-e2e --no-replicated --no-cpu-baseline --no-stream-peak > gpurun_out/bench_fp8.json 2> gpurun_out/bench_fp8.err
