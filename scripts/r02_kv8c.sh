set -x
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.txt 2>&1
timeout -k 10 300 python -m pytest tests/test_gpu_kv8.py -q -x --timeout 60 > gpurun_out/pytest_kv8.txt 2>&1
echo "rc=$?" >> gpurun_out/pytest_kv8.txt
for c in mha7b_b32_fp8 mha7b_b32; do
timeout -k 10 300 python bench.py --config $c --steps 30 --no-e2e --no-replicated --no-cpu-baseline --no-stream-peak --no-others > gpurun_out/bench_$c.json 2> gpurun_out/bench_$c.err
done
timeout -k 10 600 python scripts/timeline.py mha7b_b32_fp8 > gpurun_out/timeline8.jsonl 2> gpurun_out/timeline8.err
