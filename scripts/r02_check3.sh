# round-2 check 3: full GPU tests (fused append, FP8 KV), FP8 + C2b timing, sanitizers
set -x
mkdir -p gpurun_out/san
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.txt 2>&1
timeout 1500 python -m pytest tests -m gpu -q -x --timeout 600 -rA > gpurun_out/pytest_gpu.txt 2>&1
tail -3 gpurun_out/pytest_gpu.txt
for c in mha7b_b32_fp8 mha7b_b32; do
timeout 300 python bench.py --config $c --steps 30 --no-e2e --no-replicated --no-cpu-baseline --no-stream-peak --no-others > gpurun_out/bench_$c.json 2> gpurun_out/bench_$c.err
done
for tool in memcheck racecheck synccheck; do
  timeout 900 compute-sanitizer --tool $tool --print-limit 20 python scripts/sanitize_cases.py > gpurun_out/san/$tool.txt 2>&1
  echo "exit $?" >> gpurun_out/san/$tool.txt
done
