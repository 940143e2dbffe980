# round-1 evidence: launch list (cold, serialised) of the bench command, one
# full capture of the fused kernel (b32 and b16), and a bench line
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.txt 2>&1
B="python bench.py --steps 3 --warmup 3 --soak 0 --no-e2e --no-replicated --no-cpu-baseline"
timeout 300 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches_r01.csv $B > gpurun_out/ncu_launch.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:bif_tc_kernel -s 3 -c 1 -o gpurun_out/prof_r01_b32 $B > gpurun_out/ncu_full_b32.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:bif_tc_kernel -s 3 -c 1 -o gpurun_out/prof_r01_b16 $B --config mha7b_b16 > gpurun_out/ncu_full_b16.log 2>&1
tail -2 gpurun_out/ncu_full_b32.log gpurun_out/ncu_full_b16.log
