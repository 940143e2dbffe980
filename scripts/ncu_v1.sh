set -x
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.txt 2>&1
B="python bench.py --steps 3 --warmup 3 --soak 0 --no-e2e --no-replicated --no-cpu-baseline"
timeout 300 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/launches_v1.csv $B > /dev/null 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:ctx_tc -s 3 -c 1 -o gpurun_out/prof_ctx_v1 $B > gpurun_out/ncu_ctx.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:fma_partial -s 3 -c 1 -o gpurun_out/prof_dec_v1 $B > gpurun_out/ncu_dec.log 2>&1
ls -la gpurun_out
