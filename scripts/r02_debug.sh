set -x
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.txt 2>&1
timeout -k 5 90 python -m pytest tests/test_gpu_parity.py -q -x -k "test_small_configs or stress_variants" --timeout 30 > gpurun_out/dbg1.txt 2>&1
echo "dbg1 rc=$?" >> gpurun_out/dbg1.txt
timeout -k 5 120 python bench.py --steps 20 --no-e2e --no-replicated --no-cpu-baseline --no-stream-peak --no-others > gpurun_out/bench_mha7b_b32.json 2> gpurun_out/bench_mha7b_b32.err
timeout -k 10 900 python -m pytest tests -m gpu -q -x --timeout 60 > gpurun_out/pytest_gpu.txt 2>&1
echo "full rc=$?" >> gpurun_out/pytest_gpu.txt
