set -x
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.txt 2>&1
timeout 900 python -m pytest tests -m gpu -q -x --timeout 300 > gpurun_out/pytest_gpu.txt 2>&1
tail -5 gpurun_out/pytest_gpu.txt
timeout 300 python __graft_entry__.py smoke > gpurun_out/smoke.txt 2>&1; tail -3 gpurun_out/smoke.txt
timeout 600 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err; cat gpurun_out/bench.json; tail -5 gpurun_out/bench.err
B="python bench.py --steps 3 --warmup 3 --soak 0 --no-e2e --no-replicated --no-cpu-baseline"
timeout 600 ncu --set full --clock-control none --import-source on -k regex:bif_tc -s 3 -c 1 -o gpurun_out/prof_fused $B > gpurun_out/ncu_fused.log 2>&1
tail -3 gpurun_out/ncu_fused.log
