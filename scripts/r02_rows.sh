set -x
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.txt 2>&1
timeout -k 10 900 python -m pytest tests -m gpu -q -x --timeout 60 > gpurun_out/pytest_gpu.txt 2>&1
echo "full rc=$?" >> gpurun_out/pytest_gpu.txt
grep -E "rows: max_abs|plan-covering|b32-n4" gpurun_out/pytest_gpu.txt > gpurun_out/parity_full.txt
for c in gqa mqa long mha7b_b32 mha7b_b32_fp8; do
timeout -k 10 300 python bench.py --config $c --steps 30 --no-e2e --no-replicated --no-cpu-baseline --no-stream-peak --no-others > gpurun_out/bench_$c.json 2> gpurun_out/bench_$c.err
done
MT_CFG=mha7b_b32 timeout -k 10 300 python scripts/bench_multitoken.py > gpurun_out/mt.jsonl 2> gpurun_out/mt.err
