set -x
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.txt 2>&1
timeout 1200 python -m pytest tests -m gpu -q -x --timeout 300 --durations=15 > gpurun_out/pytest_gpu.txt 2>&1
tail -3 gpurun_out/pytest_gpu.txt
for c in mha7b_b32 mha7b_b32_fp8 mha7b_b16 gqa; do
timeout 300 python bench.py --config $c --steps 30 --no-e2e --no-replicated --no-cpu-baseline --no-stream-peak --no-others > gpurun_out/bench_$c.json 2> gpurun_out/bench_$c.err
done
timeout 600 python scripts/timeline.py mha7b_b32 mha7b_b32_fp8 > gpurun_out/timeline6.jsonl 2> gpurun_out/timeline6.err
