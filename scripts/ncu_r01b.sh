# round-1 (second session) evidence for the current kernel: launch list of the
# bench command, full captures of the fused kernel (b32 headline, gqa), bench line
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.txt 2>&1
timeout 600 python bench.py > gpurun_out/bench_r01b.json 2> gpurun_out/bench_r01b.err
B="python bench.py --steps 3 --warmup 3 --soak 0 --no-e2e --no-replicated --no-cpu-baseline"
timeout 300 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches_r01b.csv $B > gpurun_out/ncu_launch.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:bif_tc_kernel -s 3 -c 1 -o gpurun_out/prof_r01b_b32 $B > gpurun_out/ncu_full_b32.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:bif_tc_kernel -s 3 -c 1 -o gpurun_out/prof_r01b_gqa $B --config gqa > gpurun_out/ncu_full_gqa.log 2>&1
tail -2 gpurun_out/ncu_full_b32.log gpurun_out/ncu_full_gqa.log
cat gpurun_out/bench_r01b.json
