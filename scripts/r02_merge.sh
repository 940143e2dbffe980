set -x
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.txt 2>&1
timeout -k 10 900 python -m pytest tests -m gpu -q -x --timeout 60 > gpurun_out/pytest_gpu.txt 2>&1
echo "rc=$?" >> gpurun_out/pytest_gpu.txt
for c in mqa gqa long mha7b_b16 mha7b_b32; do
timeout -k 10 300 python bench.py --config $c --steps 30 --no-e2e --no-replicated --no-cpu-baseline --no-stream-peak --no-others > gpurun_out/bench_$c.json 2> gpurun_out/bench_$c.err
done
