set -x
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.txt 2>&1
timeout 600 python -m pytest tests/test_gpu_parity.py tests/test_gpu_kv8.py -q -x > gpurun_out/pytest_quick.txt 2>&1
timeout 600 python scripts/timeline.py mha7b_b32 mha7b_b32_fp8 > gpurun_out/timeline4.jsonl 2> gpurun_out/timeline4.err
for c in mha7b_b32 mha7b_b32_fp8 mha7b_b16; do
timeout 300 python bench.py --config $c --steps 30 --no-e2e --no-replicated --no-cpu-baseline --no-stream-peak --no-others > gpurun_out/bench_$c.json 2> gpurun_out/bench_$c.err
done
