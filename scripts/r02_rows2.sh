set -x
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.txt 2>&1
timeout -k 10 600 python -m pytest tests/test_gpu_parity.py tests/test_gpu_multitoken.py tests/test_gpu_append.py -q -x --timeout 60 > gpurun_out/pytest_rows.txt 2>&1
echo "rc=$?" >> gpurun_out/pytest_rows.txt
timeout -k 10 600 python scripts/role_cycles_rows.py mqa gqa > gpurun_out/role_rows2.jsonl 2> gpurun_out/role_rows2.err
for c in mqa gqa long; do
timeout -k 10 300 python bench.py --config $c --steps 30 --no-e2e --no-replicated --no-cpu-baseline --no-stream-peak --no-others > gpurun_out/bench_$c.json 2> gpurun_out/bench_$c.err
done
