# round-1 final evidence: tests, smoke, bench line, sweep, multi-token, launch list, ncu captures
set -x
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.txt 2>&1
timeout 900 python -m pytest tests -m gpu -q -x --timeout 300 > gpurun_out/pytest_gpu.txt 2>&1
tail -2 gpurun_out/pytest_gpu.txt
timeout 300 python __graft_entry__.py smoke > gpurun_out/smoke.txt 2>&1; tail -4 gpurun_out/smoke.txt
timeout 600 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err; cat gpurun_out/bench.json
bash scripts/sweep.sh
timeout 300 python scripts/bench_multitoken.py > gpurun_out/mt.jsonl 2>&1
B="python bench.py --steps 3 --warmup 3 --soak 0 --no-e2e --no-replicated --no-cpu-baseline"
timeout 300 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches_final.csv $B > gpurun_out/ncu_launch.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:bif_tc_kernel -s 3 -c 1 -o gpurun_out/prof_final_b32 $B > gpurun_out/ncu_full_b32.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:ctx_rows -s 3 -c 1 -o gpurun_out/prof_final_rows_mqa $B --config mqa > gpurun_out/ncu_rows_mqa.log 2>&1
ls gpurun_out
