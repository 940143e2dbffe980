mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.txt 2>&1
B="python bench.py --steps 3 --warmup 3 --soak 0 --no-e2e --no-replicated --no-cpu-baseline"
timeout 600 ncu --set full --clock-control none --import-source on -k regex:ctx_rows -s 3 -c 1 -o gpurun_out/prof_final_rows_gqa $B --config gqa > gpurun_out/ncu_rows_gqa.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:ctx_rows -s 3 -c 1 -o gpurun_out/prof_final_rows_mqa2 $B --config mqa > gpurun_out/ncu_rows_mqa.log 2>&1
timeout 300 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -c 100 --csv --log-file gpurun_out/launches_gqa.csv $B --config gqa > /dev/null 2>&1
for c in gqa mqa long; do timeout 300 python bench.py --config $c --steps 10 --warmup 3 --no-e2e --no-cpu-baseline --no-replicated 2>/dev/null | tail -1; done > gpurun_out/bench_cfgs.jsonl
ls gpurun_out
